"""CPU stand-in for the per-rank CUDA plan, built on the oracle (TEST ONLY).

Implements the plan methods `distributed.decompose_sharded` drives
(sharded_begin / select_local / apply_step / sharded_finish) with the CPU
oracle, so the multi-rank host logic (shard bounds, candidate all-gather,
rank-major merge, step loop) runs under gloo on the build box.  Candidates
use the same 32-byte layout and first-maximum merge as the device.
"""

import numpy as np
import torch

import oracle as O

CAND = np.dtype([("mag2", "f8"), ("flat", "i8"), ("re", "f8"), ("im", "f8")])
STEP = np.dtype([("s", "i8"), ("j", "i8"), ("radius", "f8"), ("a_re", "f8"), ("a_im", "f8"),
                 ("c_re", "f8"), ("c_im", "f8"), ("residual", "f8"), ("flags", "i4"),
                 ("margin", "f4")])


class OraclePlan:
    def __init__(self, radii, n, batch, m0, m1, device=None):
        self.radii = np.array(radii, dtype=np.float64)
        self.n, self.m0, self.m1 = n, m0, m1
        self.device = torch.device("cpu")
        self.z = O.circle(n)

    def sharded_begin(self, g):
        self.rem = [np.array(x) for x in g.numpy()]
        self.initial = [O.energy(x) for x in self.rem]
        self.stopped = [e == 0.0 for e in self.initial]
        self.nsteps = [0] * len(self.rem)

    def select_local(self, k, dc_first, batch):
        out = np.zeros(batch, CAND)
        for b in range(batch):
            if (k == 0 and dc_first) or self.stopped[b]:
                out[b] = (-1.0, np.iinfo(np.int64).max, 0.0, 0.0)
                continue
            c = O.field_argmax(O.dft_forward(self.rem[b]), self.radii, self.m0, self.m1)
            out[b] = (c["mag"], c["flat"], c["re"], c["im"])
        return torch.from_numpy(out.view(np.uint8).reshape(batch, 32).copy())

    def apply_step(self, k, max_terms, threshold, dc_first, cands, steps):
        c = cands.numpy().reshape(cands.shape[0], cands.shape[1], 32)
        for b in range(c.shape[0]):
            if self.stopped[b]:
                continue
            if k == 0 and dc_first:
                s = j = 0
                a, coeff = 0j, O.cmean(self.rem[b])
            else:
                cs = c[b].copy().view(CAND)[:, 0]
                best = max(range(len(cs)), key=lambda i: (cs[i]["mag2"], -cs[i]["flat"]))
                s, j = divmod(int(cs[best]["flat"]), self.n)
                r = self.radii[s]
                a = complex(r * self.z[j].real, r * self.z[j].imag)
                coeff = complex(cs[best]["re"], cs[best]["im"])
            self.rem[b] = O.remainder_update(self.rem[b], a, coeff)
            e = O.energy(self.rem[b])
            rec = np.zeros(1, STEP)
            rec[0] = (s, j, self.radii[s] if not (k == 0 and dc_first) else 0.0, a.real, a.imag,
                      coeff.real, coeff.imag, e, 0, 0)
            steps[b, k] = torch.from_numpy(rec.view(np.uint8).copy())
            self.nsteps[b] = k + 1
            if (threshold is not None and e <= threshold * self.initial[b]) or e == 0.0 \
                    or k + 1 >= max_terms:
                self.stopped[b] = True

    def sharded_finish(self, batch):
        return (torch.tensor(self.nsteps, dtype=torch.int32),
                torch.tensor(self.initial, dtype=torch.float64),
                torch.from_numpy(np.stack(self.rem)), torch.tensor(self.stopped, dtype=torch.int32))
