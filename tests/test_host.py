"""CPU-side checks: the C-ABI library, host validation, workload generators.

No kernel is launched here (the build box has no GPU).
"""

import ctypes as C
import os
import re
import warnings

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "afd_capi.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(afd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1711_08604_b200 import _capi
    from paper_1711_08604_b200 import build as b
    b.build()
    lib = C.CDLL(_capi.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _capi.SIGNATURES}
    assert set(declared) == bound, set(declared) ^ bound
    lib.afd_version.restype = C.c_int
    assert lib.afd_version() == 1


def test_library_is_sm100a():
    from paper_1711_08604_b200 import _capi
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_grid_and_range_validation():
    from paper_1711_08604_b200 import core
    assert core.radius_range(0.0, 0.1, 0.8) == tuple(k * 0.1 for k in range(9))
    assert len(core.radius_range(0.1, 0.1, 0.9)) == 9
    with pytest.raises(ValueError):
        core.radius_range(0.0, 0.0, 0.5)
    with pytest.raises(ValueError):
        core.radius_range(0.5, 0.1, 0.2)
    with pytest.raises(ValueError):
        core.ParameterGrid((0.5, 0.3), 64)
    with pytest.raises(ValueError):
        core.ParameterGrid((0.5, 1.0), 64)
    with pytest.raises(ValueError):
        core.ParameterGrid((), 64)
    with pytest.raises(ValueError):
        core.ParameterGrid((0.5,), 48)
    with pytest.warns(UserWarning):
        core.ParameterGrid((0.5, 0.97), 64)
    g = core.ParameterGrid.experiment_default(64)
    p = g.point(3, 16)
    assert p.radius == g.radii[3] and p.angle_index == 16
    assert core.ParameterGrid.evenly_spaced(4, 64).radii == (0.2, 0.4, 0.6, 0.8)
    with pytest.raises(ValueError):
        core.ParameterPoint(1.0, 0, 1.0 + 0j)


def test_decompose_argument_validation_before_device():
    """ValueErrors are raised on the host, exactly where the reference raises."""
    from paper_1711_08604_b200 import core
    n = 32
    g = np.ones(n, complex)
    grid = core.ParameterGrid((0.0, 0.3, 0.6), n)
    for kw in (dict(grid=core.ParameterGrid((0.0, 0.3), 64)), dict(max_terms=0),
               dict(engine="fastest"), dict(threshold=0.0), dict(threshold=1.5)):
        args = dict(grid=grid)
        args.update(kw)
        with pytest.raises(ValueError):
            core.decompose(g, **args)
    with pytest.raises(ValueError):
        core.decompose(np.full(n, np.nan + 0j), grid)
    with pytest.raises(ValueError):
        core.decompose(np.ones(12, complex), grid)
    with pytest.raises(NotImplementedError):
        core.decompose(np.ones(16384, complex), core.ParameterGrid((0.0,), 16384),
                       engine="direct")


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product raises instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1711_08604_b200 import _capi, core
    with pytest.raises(_capi.AfdCudaUnavailable):
        core.discrete_energy(np.ones(16, complex))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1711_08604_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert not re.search(r'#include\s*[<"].*oracle', src), f
                assert "libafd_oracle" not in src, f


def test_workload_shapes():
    from paper_1711_08604_b200 import workloads as W
    warnings.simplefilter("ignore")
    for name, w in W.CONFIGS.items():
        r = W.radii_for(w.m)
        assert len(r) == w.m and r[0] == 0.0 and all(b > a for a, b in zip(r, r[1:]))
    g = W.signal_for("c0")
    assert g.shape == (1024,) and g.dtype == np.complex128
    x = W.signal_for(W.CONFIGS["c2"]._replace(n=1024) if hasattr(W.CONFIGS["c2"], "_replace")
                     else W.Workload("c2s", 1024, 8, 1, 0, 0.0, 2, real=True))
    assert x.dtype == np.float64


def test_bench_arms_share_config_and_spawn(monkeypatch):
    """Both bench arms print the same `config`; --gpus N outside torchrun
    re-launches under torch.distributed.run with N ranks on 127.0.0.1."""
    import importlib
    import sys
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    from paper_1711_08604_b200 import workloads as W

    class A:
        shard, mode, gpus = "auto", "fast", 1
    w = W.CONFIGS["c4"]
    assert bench.config_dict(A, w, 1) == bench.config_dict(A, w, 1)
    assert bench.shard_mode(A, w, 1) == "single" and bench.shard_mode(A, w, 8) == "radii"
    assert bench.shard_mode(A, W.CONFIGS["c3"], 4) == "signals"
    assert bench.config_dict(A, w, 8)["parallelism"] == "dp8 over radii"
    assert bench.scaling_of("radii") == "strong" and bench.scaling_of("replicas") == "weak"
    seen = {}
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    monkeypatch.setattr(bench.os, "execv", lambda exe, cmd: seen.update(cmd=cmd))
    A.gpus = 4
    bench.maybe_spawn(A)
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4"
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_oracle_replay_detects_wrong_selection():
    """oracle.replay_check (the bench's large-grid parity): the oracle's own
    decomposition replays clean; a moved selection or a perturbed
    coefficient is caught (bitwise mode), a 1e-15 perturbation passes at
    rtol 1e-9."""
    import oracle as O
    from paper_1711_08604_b200 import workloads as W
    g = W.pole_sum(1024, 8, 0.9, 0)
    radii = np.array(W.radii_for(100))
    d = O.decompose(g, radii, max_terms=6)
    assert O.replay_check(g, radii, d.steps, 6)["ok"]
    st = d.steps.copy()
    st["j"][3] += 1
    assert not O.replay_check(g, radii, st, 6)["ok"]
    st = d.steps.copy()
    st["c_re"][2] *= 1 + 1e-15
    assert not O.replay_check(g, radii, st, 6)["ok"]
    assert O.replay_check(g, radii, st, 6, rtol=1e-9)["ok"]
