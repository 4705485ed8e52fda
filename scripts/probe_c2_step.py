"""A few AFD steps of BASELINE c2 (for launch lists of the large-N step loop)."""
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

w = W.CONFIGS["c2"]
plan = engine.get_plan(W.radii_for(w.m), w.n)
g = W.signal_for("c2")
p1 = engine.get_plan((0.0,), w.n)
x = p1.analytic_projection(torch.from_numpy(g.astype(np.complex128)).cuda()[None, :])
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = plan.decompose(x, steps)
torch.cuda.synchronize()
print("ok", out.host_steps()[1])
