"""Where the e2e time of core.decompose goes (host side), c1."""
import cProfile
import pstats
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import core, workloads as W  # noqa: E402

w = W.CONFIGS["c1"]
g = W.signal_for("c1")
grid = core.ParameterGrid(W.radii_for(w.m), w.n)
for _ in range(5):
    core.decompose(g, grid, max_terms=w.steps)
n = 200
t0 = time.perf_counter()
for _ in range(n):
    core.decompose(g, grid, max_terms=w.steps)
dt = (time.perf_counter() - t0) / n
print("core.decompose: %.1f us per call" % (dt * 1e6))
eng = core._engine()
plan = eng.get_plan(grid.radii, w.n, batch=1, engine=0)
sig = g[None, :]
t0 = time.perf_counter()
for _ in range(n):
    plan.decompose_host(sig, w.steps, None, False)
print("plan.decompose_host: %.1f us per call" % ((time.perf_counter() - t0) / n * 1e6))
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    core.decompose(g, grid, max_terms=w.steps)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
