"""Phase timings of the cluster step kernel from the AFD_STEP_TIMING debug build."""
import ctypes as C
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
os.environ["AFD_LIB_PATH"] = "paper_1711_08604_b200/lib/libafd_b200_timing.so"
from paper_1711_08604_b200 import engine, workloads as W, _capi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = W.CONFIGS[cfg]
plan = engine.get_plan(W.radii_for(w.m), w.n)
g = torch.from_numpy(W.signal_for(cfg)[None, :]).cuda()
for _ in range(3):
    plan.decompose(g, w.steps)
torch.cuda.synchronize()
out = np.zeros((64, 24), np.uint64)
lib = _capi.load()
lib.afd_debug_step_stamps.argtypes = [C.c_void_p]
assert lib.afd_debug_step_stamps(out.ctypes.data) == 0
names = ["start", "tables", "pdl_wait", "select", "update", "node", "csync1", "energy+rec",
         "fft_in", "fft_local", "csync2", "radix8", "csync3"]
rows = out[1:w.steps - 1].astype(np.int64)
d = np.diff(rows[:, :13], axis=1)
print("phase (ns, median over steps 1..28):")
for i in range(12):
    print("  %-12s -> %-12s %8.0f" % (names[i], names[i + 1], np.median(d[:, i])))
print("  select: pdl_wait -> cands reduced %.0f, -> a formed %.0f; update: -> kernel_norm %.0f" % (
    np.median(rows[:, 13] - rows[:, 2]), np.median(rows[:, 14] - rows[:, 2]),
    np.median(rows[:, 15] - rows[:, 3])))
print("  select detail: wait -> cand loop done %.0f -> stop tested+trigger %.0f -> argmax %.0f" % (
    np.median(rows[:, 16] - rows[:, 2]), np.median(rows[:, 17] - rows[:, 16]),
    np.median(rows[:, 13] - rows[:, 17])))
print("  total %.0f ns; gap step k start -> step k+1 start %.0f ns" %
      (np.median(rows[:, 12] - rows[:, 0]), np.median(np.diff(rows[:, 0]))))

# per-CTA start of the cluster (debug builds with afd_debug_step_cta_start)
if hasattr(lib, "afd_debug_step_cta_start"):
    cs = np.zeros((64, 16), np.uint64)
    lib.afd_debug_step_cta_start.argtypes = [C.c_void_p]
    lib.afd_debug_step_cta_start(cs.ctypes.data)
    cs = cs.astype(np.int64)[1:w.steps - 1]
    ncl = int((cs[0] != 0).sum())
    rel = cs[:, :ncl] - cs[:, :1]
    print("  cluster CTA start vs CTA 0 (ns, median over steps):", np.median(rel, axis=0).astype(int))
    print("  pdl_wait -> cluster wait done %.0f" % np.median(out[1:w.steps - 1, 18].astype(np.int64) -
                                                            out[1:w.steps - 1, 2].astype(np.int64)))
