"""Per-row phase timings of field_kernel from the AFD_FIELD_TIMING debug build.

Times one c1 field launch (after warm-up) and prints, per phase, the median
cycles over row-group leaders, plus the per-SM span.
"""
import ctypes as C
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
os.environ["AFD_LIB_PATH"] = "paper_1711_08604_b200/lib/libafd_b200_ftiming.so"
from paper_1711_08604_b200 import engine, workloads as W, _capi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = W.CONFIGS[cfg]
plan = engine.get_plan(W.radii_for(w.m), w.n)
g = torch.from_numpy(W.signal_for(cfg)[None, :]).cuda()
for _ in range(3):
    plan.decompose(g, w.steps)
torch.cuda.synchronize()
lib = _capi.load()
lib.afd_debug_field_stamps.argtypes = [C.c_void_p]
out = np.zeros((512, 2, 4, 16), np.int64)
assert lib.afd_debug_field_stamps(out.ctypes.data) == 0
ncta = int((out[:, :, 0, 0] != 0).any(axis=1).sum())
st = out[:ncta]
names = {2: "prologue", 3: "pass0", 4: "exch1", 5: "pass1", 6: "exch2", 7: "pass2",
         14: "epilogue"}
t0 = st[:, :, 0, 0]
print("CTAs", ncta, "  start->pdl %.0f cyc" % np.median(st[:, :, 0, 1] - t0))
for r in range(4):
    if not (st[:, :, r, 14] != 0).any():
        break
    prev = st[:, :, r - 1, 14] if r > 0 else st[:, :, 0, 1]
    row = []
    for i in (2, 3, 4, 5, 6, 7, 14):
        cur = st[:, :, r, i]
        ok = (cur != 0) & (prev != 0)
        row.append("%s %6.0f" % (names[i], np.median((cur - prev)[ok]) if ok.any() else -1))
        prev = cur
    print("row %d: " % r + "  ".join(row))
last = np.where(st[:, :, :, 14] != 0, st[:, :, :, 14], 0).max(axis=2)
span = last.max(axis=1) - t0.min(axis=1)
print("CTA span (start -> last row end): median %.0f  max %.0f cycles" % (np.median(span),
                                                                         span.max()))
d = (st[:, 0, 0, 14] - st[:, 1, 0, 14])
print("group 0 vs 1 row-0 end offset: median |d| %.0f cycles" % np.median(np.abs(d)))
