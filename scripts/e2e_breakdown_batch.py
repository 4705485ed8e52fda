"""Host-side costs inside core.decompose_batch for c3 (1024 signals; per call, ms)."""
import sys
import time
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import core, workloads as W  # noqa: E402

w = W.CONFIGS["c3"]
sig = np.stack([W.signal_for("c3", s) for s in range(w.batch)])
grid = core.ParameterGrid(W.radii_for(w.m), w.n)
core.decompose_batch(sig, grid, max_terms=w.steps)


def t(fn, n=3):
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    return (time.perf_counter() - t0) / n * 1e3, r


print("decompose_batch total %8.1f" % t(lambda: core.decompose_batch(sig, grid, max_terms=w.steps))[0])
print("validation loop      %8.1f" % t(lambda: [core._as_signal(r) for r in sig])[0])
plan = core._engine().get_plan(grid.radii, w.n, batch=w.batch, engine=0)
dt, res = t(lambda: plan.decompose_host(sig, w.steps, None, False))
print("decompose_host       %8.1f" % dt)
rec, counts, initial, rem, _, _ = res
print("_build x batch       %8.1f" % t(lambda: [core._build(grid, w.n, "fft", rec[i], int(counts[i]), initial[i], rem[i]) for i in range(w.batch)])[0])
g = torch.from_numpy(sig).cuda()
out = plan.alloc_outputs(w.batch, w.steps)
torch.cuda.synchronize()
print("device decompose     %8.1f" % t(lambda: (plan.decompose(g, w.steps, out=out), torch.cuda.synchronize()))[0])
