"""Per-step hand-off timeline (c1, or the config given as argv[1]): field and
step kernels of the last AFD step, from the AFD_FIELD_TIMING + AFD_STEP_TIMING
build (globaltimer, ns)."""
import ctypes as C
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
os.environ.setdefault("AFD_LIB_PATH", "paper_1711_08604_b200/lib/libafd_b200_both.so")
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
lib.afd_debug_step_stamps.argtypes = [C.c_void_p]
f = np.zeros((512, 2, 4, 16), np.int64)
s = np.zeros((64, 24), np.uint64)
assert lib.afd_debug_field_stamps(f.ctypes.data) == 0
assert lib.afd_debug_step_stamps(s.ctypes.data) == 0
s = s.astype(np.int64)
k = w.steps - 1
ncta = int((f[:, :, 0, 0] != 0).any(axis=1).sum())
f = f[:ncta]
t0 = s[k - 1, 12]  # step k-1 end (cluster CTA 0)
fstart = f[:, :, 0, 0]
fwait = f[:, :, 0, 1]
last = np.where(f[:, :, :, 14] != 0, f[:, :, :, 14], 0).max(axis=2)
print("times relative to the end of step k-1 (ns), k = %d" % k)
print("  field CTAs start: min %d max %d" % (fstart.min() - t0, fstart.max() - t0))
print("  field PDL wait returns: min %d median %d max %d" % (fwait.min() - t0, np.median(fwait) - t0, fwait.max() - t0))
print("  field CTAs last row done: min %d median %d max %d" % (last.min() - t0, np.median(last) - t0, last.max() - t0))
print("  step k start %d, wait returns %d, end %d" % (s[k, 0] - t0, s[k, 2] - t0, s[k, 12] - t0))
print("  step k-1: start %d wait %d (rel. to its own end: %d %d)" % (s[k-1, 0] - t0, s[k-1, 2] - t0, s[k-1,0]-s[k-1,12], s[k-1,2]-s[k-1,12]))
if os.environ.get("AFD_FLAGS"):
    print("  step k-1 signal: syncthreads %d, after signal %d" % (s[k-1, 18] - t0, s[k-1, 19] - t0))
    print("  field poll start: median %d; poll done: min %d median %d max %d" % (
        np.median(f[:, :, 0, 12]) - t0, f[:, :, 0, 13].min() - t0, np.median(f[:, :, 0, 13]) - t0,
        f[:, :, 0, 13].max() - t0))
# per-CTA spread: wait return vs end, by SM id
smid = f[:, 0, 0, 15]
wr = fwait.min(axis=1) - t0
en = last.max(axis=1) - t0
dur = en - wr
print("  per-CTA post-wait duration: min %d median %d max %d" % (dur.min(), np.median(dur), dur.max()))
print("  corr(wait return, end) = %.2f" % np.corrcoef(wr, en)[0, 1])
order = np.argsort(en)[-8:]
print("  latest CTAs (cta, smid, wait, end, dur):")
for i in order:
    print("    %3d %3d %6d %6d %6d" % (i, smid[i], wr[i], en[i], dur[i]))
lo = smid < 74
print("  SM id < 74: median end %d (n=%d); >= 74: median end %d (n=%d)" % (
    np.median(en[lo]), lo.sum(), np.median(en[~lo]), (~lo).sum()))
# per-row durations of group leaders
rowdur = f[:, :, 1, 14] - f[:, :, 0, 14]
print("  row-1 duration (ns): median %d p90 %d max %d" % (np.median(rowdur), np.percentile(rowdur, 90), rowdur.max()))
