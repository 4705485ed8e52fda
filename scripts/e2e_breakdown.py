"""Host-side costs inside core.decompose for c1 (per call, microseconds)."""
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
n = 300


def t(fn):
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    return (time.perf_counter() - t0) / n * 1e6, r


eng = core._engine()
print("decompose total      %7.1f" % t(lambda: core.decompose(g, grid, max_terms=w.steps))[0])
print("_as_signal           %7.1f" % t(lambda: core._as_signal(g))[0])
print("_check_args          %7.1f" % t(lambda: core._check_decompose_args(g[None, :], grid, 30, None, "fft"))[0])
print("get_plan             %7.1f" % t(lambda: eng.get_plan(grid.radii, w.n, batch=1, engine=0))[0])
plan = eng.get_plan(grid.radii, w.n, batch=1, engine=0)
sig = g[None, :]
dt, res = t(lambda: plan.decompose_host(sig, w.steps, None, False))
print("decompose_host       %7.1f" % dt)
rec, counts, initial, rem, _, _ = res
print("_build               %7.1f" % t(lambda: core._build(grid, w.n, "fft", rec[0], int(counts[0]), initial[0], rem[0]))[0])
