"""Field launch time vs CTAs per signal (AFD_FIELD_CTAS) at N=4096, M=1024."""
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine  # noqa: E402

b = int(sys.argv[1])
n, m = 4096, 1024
plan = engine.Plan(tuple(i / m for i in range(m)), n, max_batch=b)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).cuda()
gh = plan.dft_forward(x)
plan.time_field(gh, reps=2)
ms = plan.time_field(gh, reps=5)
tf = b * m * n * 67 / (ms * 1e-3) / 1e12
print("batch=%d ctas/signal=%s  %.3f ms  %.2f TF/s  frac %.3f" % (
    b, os.environ.get("AFD_FIELD_CTAS", "auto"), ms, tf, tf / engine.fp64_peak_tflops()))
