"""One field launch at (N, M, batch) for profiling."""
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

n, m, b = (int(a) for a in sys.argv[1:4])
plan = engine.get_plan(W.radii_for(m), n, batch=b)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).cuda()
gh = plan.dft_forward(x)
ms = plan.time_field(gh, reps=2)
print("N=%d M=%d batch=%d field %.3f ms" % (n, m, b, ms))
