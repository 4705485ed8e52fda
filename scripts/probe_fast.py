"""Field launch time, exact vs fast mode: python scripts/probe_fast.py N M BATCH FAST [REPS].

Prints ms per field evaluation (all rows, all signals), evals/s, credited
TFLOP/s (F(N) = 5 log2 N + 7 per eval) and, for N > 8192, GB/s at the
algorithmic bytes (32 B/eval fast; exact adds the live r^l table)."""
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

n, m, b, fast = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
plan = engine.Plan(W.radii_for(m), n, max_batch=b, fast=fast)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).cuda()
gh = plan.dft_forward(x)
plan.time_field(gh, reps=1)
ms = plan.time_field(gh, reps=reps)
ev = b * m * n
tf = ev * (5 * (n.bit_length() - 1) + 7) / (ms * 1e-3) / 1e12
extra = ""
if n > 8192:
    extra = "  %.0f GB/s at 32 B/eval" % (ev * 32 / (ms * 1e-3) / 1e9)
print("N=%d M=%d batch=%d fast=%d  field %.4f ms  %.3e evals/s  %.2f TF/s%s"
      % (n, m, b, fast, ms, ev / (ms * 1e-3), tf, extra), flush=True)
