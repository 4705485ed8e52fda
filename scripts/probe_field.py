"""Field-kernel throughput probe: TFLOP/s (F(N) = 5 log2 N + 7 per eval) vs launch size."""
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

peak = engine.fp64_peak_tflops()
print("fp64 peak %.2f TF/s" % peak)
for n, m, b in [(4096, 512, 1), (4096, 1024, 1), (4096, 1024, 8), (4096, 1024, 64),
                (1024, 100, 1), (1024, 1024, 16), (8192, 1024, 4), (256, 1024, 64)]:
    radii = W.radii_for(m)
    plan = engine.get_plan(radii, n, batch=b)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).cuda()
    gh = plan.dft_forward(x)
    plan.time_field(gh, reps=3)
    ms = plan.time_field(gh, reps=10)
    ev = b * m * n
    tf = ev * (5 * (n.bit_length() - 1) + 7) / (ms * 1e-3) / 1e12
    print("N=%5d M=%5d batch=%3d  %.3f ms  %.3e evals/s  %.2f TF/s  %.1f%% of peak"
          % (n, m, b, ms, ev / (ms * 1e-3), tf, 100 * tf / peak))
