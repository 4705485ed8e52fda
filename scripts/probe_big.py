"""Large-N field probe (one c2-sized field evaluation, M=4096 radii, N=65536)."""
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
plan = engine.get_plan(W.radii_for(m), n)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal(n) + 1j * rng.standard_normal(n)).cuda()
gh = plan.dft_forward(x)
ms = plan.time_field(gh, reps=reps)
ev = m * n
tf = ev * (5 * (n.bit_length() - 1) + 7) / (ms * 1e-3) / 1e12
print("N=%d M=%d field %.3f ms  %.3e evals/s  %.2f TF/s" % (n, m, ms, ev / (ms * 1e-3), tf))
