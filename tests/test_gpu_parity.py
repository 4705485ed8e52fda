"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Every comparison is exact (np.array_equal: bitwise up to the sign of zero):
the device kernels reproduce the reference's numpy arithmetic operation for
operation.  All calls go through the C ABI (libafd_b200.so) via the
package's public API.
"""

import json
import os
import warnings

import numpy as np
import pytest

import oracle as O
from conftest import DECOMP_CASES, ROOT, load_golden

pytestmark = pytest.mark.gpu

warnings.simplefilter("ignore", UserWarning)


@pytest.fixture(scope="module")
def afd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1711_08604_b200 import core, engine
    return core, engine


@pytest.fixture(scope="module")
def tr():
    return load_golden("transforms.npz")


ONCHIP = [8, 16, 64, 256, 1024, 4096, 8192]


@pytest.mark.parametrize("n", ONCHIP)
def test_transforms_bitwise(afd, tr, n):
    core, engine = afd
    from paper_1711_08604_b200 import transform
    x = tr["x_%d" % n]
    assert np.array_equal(transform.dft_forward(x), tr["fwd_%d" % n])
    assert np.array_equal(transform.dft_inverse(x), tr["inv_%d" % n])
    c = tr["fwd_%d" % n]
    radii = tuple(tr["radii_%d" % n])
    assert np.array_equal(transform.weighted_inverse_grid(c, radii), tr["field_%d" % n])
    assert core.discrete_energy(x) == tr["energy_%d" % n]
    assert np.array_equal(core.analytic_projection(tr["xr_%d" % n]), tr["proj_%d" % n])
    a, cc = complex(tr["a_%d" % n]), complex(tr["c_%d" % n])
    assert np.array_equal(core.kernel_samples(a, n), tr["ks_%d" % n])
    assert np.array_equal(core.blaschke_samples(a, n), tr["bs_%d" % n])
    assert np.array_equal(core.remainder_update(x, a, cc), tr["upd_%d" % n])


def _check_decomp(d, g, bitwise=True):
    assert len(d.steps) == len(g["j"])
    for k, s in enumerate(d.steps):
        assert s.point.angle_index == g["j"][k], k
        assert s.point.radius == g["radius"][k], k
        assert s.point.value == g["a"][k], k
        if bitwise:
            assert s.coefficient == g["coeff"][k], k
            assert s.residual_energy == g["residual"][k], k
        else:
            assert abs(s.coefficient - g["coeff"][k]) <= 1e-9 * abs(g["coeff"][k])
    assert d.initial_energy == g["initial"]
    if bitwise:
        assert np.array_equal(d.remainder, g["remainder"])


@pytest.mark.parametrize("case", [c for c in DECOMP_CASES if c != "big16384"])
def test_decompose_matches_reference(afd, case):
    core, _ = afd
    g = load_golden("decomp_%s.npz" % case)
    thr = float(g["threshold"])
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    d = core.decompose(g["g"], grid, max_terms=int(g["max_terms"]),
                       threshold=None if np.isnan(thr) else thr, dc_first=bool(g["dc_first"]))
    _check_decomp(d, g)
    if d.steps:
        assert np.array_equal(np.array(core.error_trace(d, g["g"])), g["trace"])
        assert np.array_equal(core.reconstruct(d, len(d.steps)), g["reconstruction"])


def test_decompose_batch_equals_single(afd):
    """c3-style batch: entry b equals the single-signal decomposition."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    g0 = load_golden("decomp_c3_s0.npz")
    g1 = load_golden("decomp_c3_s1.npz")
    w = W.CONFIGS["c3"]
    sigs = np.stack([g0["g"], g1["g"], W.signal_for("c3", 2), np.zeros(w.n, complex)])
    grid = core.ParameterGrid(W.radii_for(w.m), w.n)
    ds = core.decompose_batch(sigs, grid, max_terms=w.steps)
    _check_decomp(ds[0], g0)
    _check_decomp(ds[1], g1)
    single = core.decompose(sigs[2], grid, max_terms=w.steps)
    assert [s.point for s in ds[2].steps] == [s.point for s in single.steps]
    assert np.array_equal(ds[2].remainder, single.remainder)
    assert len(ds[3].steps) == 0 and ds[3].initial_energy == 0.0


@pytest.mark.parametrize("n,m", [(64, 7), (1024, 100), (4096, 33)])
def test_field_argmax_matches_oracle(afd, n, m):
    _, engine = afd
    import torch
    rng = np.random.Generator(np.random.Philox(n + m))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    radii = tuple(np.sort(rng.uniform(0, 0.99, m)))
    plan = engine.get_plan(radii, n)
    gh = plan.dft_forward(torch.from_numpy(x).cuda())
    cand = plan.field_argmax(gh).cpu().numpy().view(
        np.dtype([("mag2", "f8"), ("flat", "i8"), ("re", "f8"), ("im", "f8")]))[0, 0]
    ref = O.field_argmax(O.dft_forward(x), np.array(radii))
    assert int(cand["flat"]) == int(ref["flat"])
    assert cand["mag2"] == ref["mag"] and cand["re"] == ref["re"] and cand["im"] == ref["im"]


def test_single_atom_recovery(afd):
    """Reference acceptance criterion 6 (test_acceptance.py:118-132)."""
    core, _ = afd
    n = 256
    grid = core.ParameterGrid.experiment_default(n)
    target = grid.point(5, 17)
    g = core.kernel_samples(target, n)
    d = core.decompose(g, grid, max_terms=1)
    st = d.steps[0]
    assert (st.point.radius, st.point.angle_index) == (target.radius, target.angle_index)
    assert st.point.value == target.value
    assert st.residual_energy < 1e-10 * d.initial_energy


def test_zero_and_constant_signals(afd):
    core, _ = afd
    n = 32
    grid = core.ParameterGrid((0.0, 0.3, 0.6), n)
    d = core.decompose(np.zeros(n, complex), grid)
    assert len(d) == 0 and d.initial_energy == 0.0 and np.array_equal(d.remainder, np.zeros(n))
    d = core.decompose(np.full(n, 2.0 + 1.0j), grid, max_terms=5)
    assert len(d) == 1 and d.steps[0].point.value == 0j and d.steps[0].residual_energy == 0.0


def test_maximal_selection_tie_breaks_row_major(afd):
    core, _ = afd
    grid = core.ParameterGrid((0.0, 0.2, 0.4), 8)
    f = np.zeros((3, 8), dtype=np.complex128)
    f[1, 3] = 2.0
    f[2, 0] = -2.0
    point, coeff = core.maximal_selection(f, grid)
    assert (point.radius, point.angle_index) == (0.2, 3) and coeff == 2.0


def test_tm_basis_and_relative_error(afd):
    core, _ = afd
    g = load_golden("decomp_f1_dc.npz")
    n = g["g"].shape[0]
    poles = list(g["a"][:4])
    b = core.tm_basis_samples(poles, n)
    ref = O.kernel_samples(poles[-1], n)
    for a in poles[:-1]:
        ref = ref * O.blaschke_samples(a, n)
    assert np.array_equal(b, ref)
    s = g["reconstruction"]
    assert core.relative_error(g["g"], s) == g["trace"][-1]


def test_launch_count_advances(afd):
    """The hot path runs this library's kernels (no silent fallback)."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c0"]
    radii = W.radii_for(w.m)
    plan = engine.get_plan(radii, w.n)
    before = plan.launch_count()
    core.decompose(W.signal_for("c0"), core.ParameterGrid(radii, w.n), max_terms=w.steps)
    assert plan.launch_count() - before >= 1 + 2 * w.steps


# ---------------------------------------------------------------------------
# large N (two-level DIT, afd_big.cuh)
# ---------------------------------------------------------------------------

def _big_input(n, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


@pytest.mark.parametrize("n", [16384, 65536, 1 << 20])
def test_big_n_transforms_bitwise(afd, n):
    core, _ = afd
    from paper_1711_08604_b200 import transform
    b = load_golden("big.npz")
    x = _big_input(n, n)
    sel = np.arange(0, n, 4099) if n > 16384 else np.arange(n)
    a, c = complex(b["a_%d" % n]), complex(b["c_%d" % n])
    fwd = transform.dft_forward(x)
    assert np.array_equal(fwd[sel], b["fwd_%d" % n])
    assert np.array_equal(transform.dft_inverse(x)[sel], b["inv_%d" % n])
    assert np.array_equal(core.kernel_samples(a, n)[sel], b["ks_%d" % n])
    assert np.array_equal(core.blaschke_samples(a, n)[sel], b["bs_%d" % n])
    upd = core.remainder_update(x, a, c)
    assert np.array_equal(upd[sel], b["upd_%d" % n])
    assert core.discrete_energy(x) == b["energy_%d" % n]
    assert core.discrete_energy(upd) == b["upd_energy_%d" % n]
    if n <= 65536:
        f = transform.weighted_inverse_grid(fwd, tuple(b["radii_%d" % n]))
        assert np.array_equal(f[:, sel], b["field_%d" % n])


def test_big_n_decompose_matches_reference(afd):
    core, _ = afd
    g = load_golden("decomp_big16384.npz")
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    d = core.decompose(g["g"], grid, max_terms=int(g["max_terms"]))
    _check_decomp(d, g)
    assert np.array_equal(np.array(core.error_trace(d, g["g"])), g["trace"])


def test_c2_projection_and_first_steps(afd):
    """BASELINE c2 (N=65536, M=4096, real input): projection + 2 AFD steps."""
    core, _ = afd
    g = load_golden("c2_step.npz")
    proj = core.analytic_projection(g["x"])
    assert np.array_equal(proj, g["g"])
    grid = core.ParameterGrid(tuple(g["radii"]), proj.shape[0])
    d = core.decompose(proj, grid, max_terms=len(g["s"]))
    for k, st in enumerate(d.steps):
        assert grid.radii.index(st.point.radius) == g["s"][k]
        assert st.point.angle_index == g["j"][k]
        assert st.coefficient == g["coeff"][k]
        assert st.residual_energy == g["residual"][k]
    assert d.initial_energy == g["initial"]
    assert np.array_equal(d.remainder, g["remainder"])


def test_c4_length_decompose_matches_oracle(afd):
    """N = 2^20 (c4's length) on a small radius grid vs the CPU oracle."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << 20
    g = W.pole_sum(n, 128, 0.99, 4)
    radii = (0.0, 0.5, 0.9, 0.99, 0.999)
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=3)
    o = O.decompose(g, np.array(radii), max_terms=3)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert np.array_equal(d.remainder, o.remainder)


@pytest.mark.parametrize("m", [100, 163])
def test_field_n65536_matches_oracle(afd, m):
    """N = 2^16 (c2's length) over M = 100 / 163 radii: the large-N field
    (pass A + column pass, all rows in one batch) — selections, coefficients,
    energies and remainder vs the oracle."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << 16
    g = W.pole_sum(n, 32, 0.97, 7)
    radii = tuple(i / m for i in range(m))
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=3)
    o = O.decompose(g, np.array(radii), max_terms=3)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert np.array_equal(d.remainder, o.remainder)


@pytest.mark.parametrize("k,m", [(15, 40), (21, 3), (22, 2)])
def test_large_n_column_pass_lengths_match_oracle(afd, k, m):
    """N = 2^15 (pass A of 2^11 points + the 4-stage TMA column pass) and
    N = 2^21 / 2^22 (pass A of 2^9 / 2^10, an in-place 8-stage column pass,
    then the 4-stage TMA column pass): decomposition vs the CPU oracle."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 16, 0.97, k)
    radii = tuple(0.999 * i / m for i in range(m))
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=2)
    o = O.decompose(g, np.array(radii), max_terms=2)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert np.array_equal(d.remainder, o.remainder)


@pytest.mark.parametrize("k", [16, 18])
def test_large_n_multi_batch_matches_oracle(afd, k, monkeypatch):
    """Row batches forced to 2 rows (AFD_BIG_ROWS, read at plan creation):
    7 radii = 4 batches, the last one partial, through the block-major pass A
    and the TMA column pass (N = 2^18: tensor map over 2-row batches)."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    monkeypatch.setenv("AFD_BIG_ROWS", "2")
    n = 1 << k
    g = W.pole_sum(n, 16, 0.96, 300 + k)
    radii = tuple(0.997 * i / 7 for i in range(7))
    plan = engine.Plan(radii, n, max_batch=1)  # private plan: built with 2-row batches
    rec, counts, initial, rem, _, _ = plan.decompose_host(g[None, :], 3)
    o = O.decompose(g, np.array(radii), max_terms=3)
    c = int(counts[0])
    assert c == len(o.steps)
    assert np.array_equal(rec[0]["j"][:c], o.steps["j"])
    assert np.array_equal(rec[0]["radius"][:c], o.steps["radius"])
    assert np.array_equal(rec[0]["c_re"][:c], o.steps["c_re"])
    assert np.array_equal(rec[0]["c_im"][:c], o.steps["c_im"])
    assert np.array_equal(rec[0]["residual"][:c], o.steps["residual"])
    assert np.array_equal(rem[0], o.remainder)


def test_c4_full_size_first_step(afd):
    """BASELINE c4 at full size (N = 2^20, M = 16384: a 128 GiB r^l table, 74
    row batches), first AFD step on the GPU.  The oracle cannot evaluate the
    whole 2^34-point grid here, so the check is row-local: the selected point
    is, bit for bit, the first maximum of its own row as the oracle computes
    it; no row of a seeded sample (plus the neighbours) beats it under the
    reference's order; the coefficient, remainder and energy equal the
    oracle's update with that atom."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c4"]
    g = W.signal_for("c4")
    radii = np.array(W.radii_for(w.m))
    plan = engine.Plan(tuple(radii), w.n, max_batch=1)
    try:
        rec, counts, initial, rem, _, _ = plan.decompose_host(g[None, :], 1)
    finally:
        del plan
    r = rec[0][0]
    s, j = int(r["s"]), int(r["j"])
    flat = s * w.n + j
    ghat = O.dft_forward(g)
    own = O.field_argmax(ghat, radii, s, s + 1)
    assert int(own["flat"]) == flat
    assert own["re"] == r["c_re"] and own["im"] == r["c_im"]
    rng = np.random.default_rng(44)
    rows = sorted(set(rng.integers(0, w.m, 20).tolist()) | {max(s - 1, 0), min(s + 1, w.m - 1),
                                                            w.m - 1})
    for row in rows:
        c = O.field_argmax(ghat, radii, row, row + 1)
        assert c["mag"] < own["mag"] or (c["mag"] == own["mag"] and c["flat"] >= flat), row
    a = complex(r["a_re"], r["a_im"])
    want = O.remainder_update(g, a, complex(r["c_re"], r["c_im"]))
    assert np.array_equal(rem[0], want)
    assert r["residual"] == O.energy(want)


@pytest.mark.parametrize("k,dc,thr", [(14, True, None), (16, True, 0.3), (18, False, 0.6)])
def test_large_n_dc_first_and_threshold(afd, k, dc, thr):
    """Large N with the numpy-mean atom first (pairwise complex sum over N on
    the device) and/or the energy-threshold stop, vs the oracle."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 12, 0.95, 400 + k) + 0.25
    radii = tuple(0.99 * i / 6 for i in range(6))
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=5, threshold=thr,
                       dc_first=dc)
    o = O.decompose(g, np.array(radii), max_terms=5, threshold=thr, dc_first=dc)
    assert len(d.steps) == len(o.steps)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert np.array_equal(d.remainder, o.remainder)


@pytest.mark.parametrize("k", [17, 18, 19])
def test_fused_column_pass_lengths_match_oracle(afd, k):
    """N = 2^17..2^19: pass A of 2^9..2^11 points then the 8-stage fused
    column pass (big_pass_col8), field argmax + update vs the CPU oracle."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 24, 0.97, k)
    radii = (0.0, 0.3, 0.7, 0.9, 0.97, 0.995)
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=3)
    o = O.decompose(g, np.array(radii), max_terms=3)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert np.array_equal(d.remainder, o.remainder)


@pytest.mark.parametrize("case", ["c0", "f2_dc", "big16384"])
def test_sharded_step_api_on_one_gpu(afd, case):
    """Two radius shards driven through afd_select_local / afd_apply_step,
    with the all-gather emulated by concatenation (no cross-rank waiting),
    reproduce the reference decomposition exactly."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import _capi
    from paper_1711_08604_b200.distributed import shard_bounds
    g = load_golden("decomp_%s.npz" % case)
    radii = tuple(g["radii"])
    n = g["g"].shape[0]
    max_terms = int(g["max_terms"])
    thr = float(g["threshold"])
    thr = None if np.isnan(thr) else thr
    dc = bool(g["dc_first"])
    world = 2
    plans = [engine.Plan(radii, n, *shard_bounds(len(radii), r, world), max_batch=1)
             for r in range(world)]
    x = torch.from_numpy(g["g"][None, :]).cuda()
    steps = [torch.zeros((1, max_terms, _capi.STEP_DTYPE.itemsize), dtype=torch.uint8,
                         device="cuda") for _ in plans]
    for p in plans:
        p.sharded_begin(x)
    for k in range(max_terms):
        local = [p.select_local(k, dc, 1) for p in plans]
        cands = torch.stack(local, 1).contiguous()
        for p, s in zip(plans, steps):
            p.apply_step(k, max_terms, thr, dc, cands, s)
    for p, s in zip(plans, steps):
        n_steps, initial, rem, _ = p.sharded_finish(1)
        count = int(n_steps.cpu()[0])
        rec = s.cpu().numpy().view(_capi.STEP_DTYPE)[0, :count, 0]
        assert count == len(g["j"])
        assert np.array_equal(rec["j"], g["j"]) and np.array_equal(rec["radius"], g["radius"])
        assert np.array_equal(rec["c_re"] + 1j * rec["c_im"], g["coeff"])
        assert np.array_equal(rec["residual"], g["residual"])
        assert np.array_equal(rem.cpu().numpy()[0], g["remainder"])


@pytest.mark.parametrize("k", [16, 18])
def test_sharded_large_n_matches_oracle(afd, k):
    """Three radius shards of a large-N grid (N = 2^16: TMA 4-stage column
    pass; 2^18: tensor-map 8-stage column pass) through afd_select_local /
    afd_apply_step with the all-gather emulated: every shard's records and
    remainder equal the CPU oracle's decomposition."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import _capi, workloads as W
    from paper_1711_08604_b200.distributed import shard_bounds
    n = 1 << k
    g = W.pole_sum(n, 20, 0.97, 100 + k)
    radii = tuple(0.998 * i / 7 for i in range(7))
    max_terms, world = 3, 3
    o = O.decompose(g, np.array(radii), max_terms=max_terms)
    plans = [engine.Plan(radii, n, *shard_bounds(len(radii), r, world), max_batch=1)
             for r in range(world)]
    x = torch.from_numpy(g[None, :]).cuda()
    steps = [torch.zeros((1, max_terms, _capi.STEP_DTYPE.itemsize), dtype=torch.uint8,
                         device="cuda") for _ in plans]
    for p in plans:
        p.sharded_begin(x)
    for kk in range(max_terms):
        cands = torch.stack([p.select_local(kk, False, 1) for p in plans], 1).contiguous()
        for p, s in zip(plans, steps):
            p.apply_step(kk, max_terms, None, False, cands, s)
    for p, s in zip(plans, steps):
        n_steps, initial, rem, _ = p.sharded_finish(1)
        count = int(n_steps.cpu()[0])
        rec = s.cpu().numpy().view(_capi.STEP_DTYPE)[0, :count, 0]
        assert count == len(o.steps)
        assert np.array_equal(rec["j"], o.steps["j"])
        assert np.array_equal(rec["radius"], o.steps["radius"])
        assert np.array_equal(rec["c_re"], o.steps["c_re"])
        assert np.array_equal(rec["c_im"], o.steps["c_im"])
        assert np.array_equal(rec["residual"], o.steps["residual"])
        assert np.array_equal(rem.cpu().numpy()[0], o.remainder)


def test_signal_sharded_batch_one_nccl_rank(afd):
    """distributed.decompose_batch_sharded on a one-rank NCCL group equals
    core.decompose_batch (the c3 multi-GPU entry point, gather included)."""
    core, _ = afd
    import socket
    import torch.distributed as dist
    from paper_1711_08604_b200 import distributed, workloads as W
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0,
                            world_size=1)
    try:
        n, radii = 1024, tuple(i / 64 for i in range(64))
        sig = np.stack([W.pole_sum(n, 8, 0.9, 200 + s) for s in range(5)])
        grid = core.ParameterGrid(radii, n)
        got = distributed.decompose_batch_sharded(sig, grid, max_terms=6)
        want = core.decompose_batch(sig, grid, max_terms=6)
        assert len(got) == len(want) == 5
        for a, b in zip(got, want):
            assert a.steps == b.steps
            assert np.array_equal(a.remainder, b.remainder)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# size-independent properties at BASELINE sizes (reference acceptance
# criteria 2, 7, 8: tests/test_acceptance.py:66-76, 135-166)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_energy_and_reconstruction_identities_at_baseline_size(afd, cfg):
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS[cfg]
    g = W.signal_for(cfg, 5)
    grid = core.ParameterGrid(W.radii_for(w.m), w.n)
    d = core.decompose(g, grid, max_terms=w.steps)
    e0 = d.initial_energy
    spent = 0.0
    for st in d.steps:                                   # criterion 2
        spent += abs(st.coefficient) ** 2
        assert abs((e0 - spent) - st.residual_energy) < 1e-10 * e0
    tail = d.remainder.copy()                            # criterion 7
    for st in d.steps:
        tail *= core.blaschke_samples(st.point, w.n)
    gap = np.max(np.abs(g - core.reconstruct(d, len(d.steps)) - tail))
    assert gap < 1e-10 * np.max(np.abs(g))
    res = [e0] + [s.residual_energy for s in d.steps]     # monotone residuals
    assert all(b <= a * (1 + 1e-12) for a, b in zip(res, res[1:]))


def test_basis_orthonormality_of_selected_poles(afd):
    """Criterion 8 on the c0 decomposition's poles (Gram deviation < 1e-9)."""
    core, _ = afd
    g = load_golden("decomp_c0.npz")
    n = g["g"].shape[0]
    poles = list(g["a"])
    basis = [core.tm_basis_samples(poles[: k + 1], n) for k in range(len(poles))]
    gram = np.array([[np.mean(bi * np.conj(bj)) for bj in basis] for bi in basis])
    assert np.max(np.abs(gram - np.eye(len(poles)))) < 1e-9


def test_parallel_flag_and_single_rows_identical(afd):
    """parallel=True is result-identical (test_core.py:175-182); single-radius
    rows equal grid rows bitwise (test_transform.py:206-213)."""
    core, _ = afd
    from paper_1711_08604_b200 import transform
    g = load_golden("decomp_rand3.npz")
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    a = core.decompose(g["g"], grid, max_terms=6)
    b = core.decompose(g["g"], grid, max_terms=6, parallel=True)
    assert [s.point for s in a.steps] == [s.point for s in b.steps]
    assert [s.coefficient for s in a.steps] == [s.coefficient for s in b.steps]
    c = transform.dft_forward(g["g"])
    rows = transform.weighted_inverse_grid(c, (0.0, 0.25, 0.5, 0.8))
    for i, r in enumerate((0.0, 0.25, 0.5, 0.8)):
        assert np.array_equal(rows[i], transform.weighted_inverse(c, r))


def test_scale_invariance_of_selection(afd):
    """test_core.py:350-360: scaling G scales coefficients, keeps poles."""
    core, _ = afd
    g = load_golden("decomp_rand11.npz")["g"]
    grid = core.ParameterGrid.experiment_default(g.shape[0])
    base = core.decompose(g, grid, max_terms=4)
    for scale in (1e-6, 137.0, 1e6):
        sc = core.decompose(scale * g, grid, max_terms=4)
        for sb, ss in zip(base.steps, sc.steps):
            assert sb.point.value == ss.point.value
            assert abs(ss.coefficient - scale * sb.coefficient) < 1e-12 * scale * abs(sb.coefficient)


def test_pow_ambiguity_flags_consistent(afd):
    """Steps flagged 'pow-ambiguous' are exactly those whose |a|*|a| low part
    exceeds 0.49 ulp; unflagged steps are provably bit-identical."""
    core, _ = afd
    import math
    g = load_golden("decomp_c1.npz")
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    d = core.decompose(g["g"], grid, max_terms=int(g["max_terms"]))
    for st, fl in zip(d.steps, d.step_flags):
        h = abs(st.point.value)
        hh = h * h
        # exact low part of h*h via Dekker's split
        sp = 134217729.0
        t = sp * h
        hi = t - (t - h)
        lo_ = h - hi
        err = ((hi * hi - hh) + 2 * hi * lo_) + lo_ * lo_
        ulp = math.ulp(hh) if hh else 0.0
        assert bool(fl & 1) == (hh != 0.0 and abs(err) > 0.49 * ulp)
        if not fl & 1:
            assert h ** 2 == hh  # CPython's pow agrees with the device's h*h


# ---------------------------------------------------------------------------
# direct engine (oracle.field_direct on the device)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["rand3", "rand11", "rand42", "c0"])
def test_direct_engine_matches_reference(afd, case):
    """engine="direct": the reference's engine-agreement contract
    (test_core.py:313-326): identical poles, coefficients and residuals to
    1e-9; field rows vs oracle.field_direct to 1e-9 (criterion 1)."""
    core, _ = afd
    from paper_1711_08604_b200 import direct
    dg = load_golden("direct.npz")
    g = dg["g_" + case]
    grid = core.ParameterGrid(tuple(dg["radii_" + case]), g.shape[0])
    f = direct.field_direct(g, grid)
    ref = dg["field_" + case]
    assert np.max(np.abs(f - ref) / np.maximum(np.abs(ref), 1e-300)) < 1e-9
    d = core.decompose(g, grid, max_terms=int(dg["terms_" + case]), engine="direct")
    assert d.engine == "direct"
    assert [s.point.angle_index for s in d.steps] == list(dg["j_" + case])
    assert [s.point.radius for s in d.steps] == list(dg["radius_" + case])
    e0 = d.initial_energy
    for st, c, r in zip(d.steps, dg["coeff_" + case], dg["residual_" + case]):
        assert abs(st.coefficient - c) < 1e-9 * abs(c)
        assert abs(st.residual_energy - r) < 1e-9 * e0
    # and the fft engine selects the same poles (test_core.py:313-326)
    d2 = core.decompose(g, grid, max_terms=int(dg["terms_" + case]), engine="fft")
    assert [s.point for s in d2.steps] == [s.point for s in d.steps]


# ---------------------------------------------------------------------------
# command line on the device: files byte-identical to the reference CLI's
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["f1_256", "f2_1024", "rand_512"])
def test_cli_outputs_byte_identical(afd, tmp_path, case):
    import os
    from conftest import GOLDEN
    from paper_1711_08604_b200 import cli
    ref = os.path.join(GOLDEN, "cli")
    dec = {"rand_512": ["--terms", "8", "--no-dc-first", "--radii", "0.05,0.3,0.55,0.8,0.9"]}
    js = tmp_path / "d.json"
    assert cli.run_command(["decompose", "--input", os.path.join(ref, case + ".csv"),
                            "--output", str(js)] + dec.get(case, ["--terms", "10"])) == 0
    assert js.read_bytes() == open(os.path.join(ref, case + ".json"), "rb").read()
    s4, err = tmp_path / "s4.csv", tmp_path / "err.csv"
    assert cli.run_command(["reconstruct", "--input", str(js), "--terms", "4", "--output",
                            str(s4), "--emit-errors", str(err)]) == 0
    assert s4.read_bytes() == open(os.path.join(ref, case + ".s4.csv"), "rb").read()
    assert err.read_bytes() == open(os.path.join(ref, case + ".err.csv"), "rb").read()
    if case == "f2_1024":  # synth f2 runs the analytic projection on the device
        sc = tmp_path / "f2.csv"
        assert cli.run_command(["synth", "f2", "--samples", "1024", "--output", str(sc)]) == 0
        assert sc.read_bytes() == open(os.path.join(ref, "f2_1024.csv"), "rb").read()


def test_cli_bench_runs(afd, tmp_path):
    from paper_1711_08604_b200 import cli
    out = tmp_path / "b.csv"
    assert cli.run_command(["bench", "--sizes", "256,512,1024", "--repeats", "2", "--output",
                            str(out)]) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "engine,N,M,terms,repeat,seconds" and len(rows) == 1 + 2 * 3 * 2
    summary = json.loads((tmp_path / "b.summary.json").read_text())
    assert set(summary["engines"]) == {"fft", "direct"}


# ---------------------------------------------------------------------------
# the N = 4096 field kernel variant with both row-groups per SM (TMEM
# twiddles and spectrum, group offset) is only launched for >= 2*SMs rows;
# these cases run it (materialised rows and argmax) against the oracle
# ---------------------------------------------------------------------------

def test_field_rows_n4096_full_grid_bitwise(afd):
    _, engine = afd
    import torch
    n, m = 4096, 320
    rng = np.random.Generator(np.random.Philox(4096 + m))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    radii = tuple(np.sort(rng.uniform(0, 0.98, m)))
    plan = engine.get_plan(radii, n)
    gh = plan.dft_forward(torch.from_numpy(x).cuda())
    rows = plan.field(gh).cpu().numpy()
    ref = O.field(O.dft_forward(x), np.array(radii))
    assert rows.shape == ref.shape
    assert np.array_equal(rows.view(np.uint64), ref.view(np.uint64))
    cand = plan.field_argmax(gh).cpu().numpy().view(
        np.dtype([("mag2", "f8"), ("flat", "i8"), ("re", "f8"), ("im", "f8")]))[0, 0]
    ref_c = O.field_argmax(O.dft_forward(x), np.array(radii))
    assert int(cand["flat"]) == int(ref_c["flat"])
    assert cand["re"] == ref_c["re"] and cand["im"] == ref_c["im"]


def test_c1_decomposition_bitwise_vs_oracle(afd):
    """The benchmark workload itself (c1: N=4096, M=512, 30 steps)."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c1"]
    g = W.signal_for("c1")
    radii = W.radii_for(w.m)
    d = core.decompose(g, core.ParameterGrid(radii, w.n), max_terms=w.steps)
    o = O.decompose(g, np.array(radii), max_terms=w.steps)
    assert len(d.steps) == len(o.steps) == w.steps
    for st, ref in zip(d.steps, o.steps):
        assert (st.point.radius, st.point.angle_index) == (ref["radius"], int(ref["j"]))
        assert st.coefficient == complex(ref["c_re"], ref["c_im"])
        assert st.residual_energy == ref["residual"]
    assert np.array_equal(d.remainder.view(np.uint64), o.remainder.view(np.uint64))


@pytest.mark.parametrize("n,m,dc,thr", [(4096, 96, True, None), (4096, 64, False, 0.02),
                                        (8192, 1100, True, 0.05), (2048, 40, True, None)])
def test_cluster_step_options_vs_oracle(afd, n, m, dc, thr):
    """dc_first / threshold through the 16-CTA cluster step kernel (N = 2048..8192; at
    N = 8192 with > 1024 radii the pole lookup reads the radii from global memory)."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    g = W.pole_sum(n, 20, 0.95, n + m)
    radii = tuple(k / m for k in range(m))
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=12, threshold=thr,
                       dc_first=dc)
    o = O.decompose(g, np.array(radii), max_terms=12, threshold=thr, dc_first=dc)
    assert len(d.steps) == len(o.steps)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    assert [s.coefficient for s in d.steps] == list(o.steps["c_re"] + 1j * o.steps["c_im"])
    assert [s.residual_energy for s in d.steps] == list(o.steps["residual"])
    assert d.initial_energy == o.initial_energy
    assert np.array_equal(d.remainder.view(np.uint64), o.remainder.view(np.uint64))


def test_bench_line_contract(afd):
    """bench.py's default JSON line (the driver's command, shortened): the
    contract keys, the required workload (c4, the largest one-GPU config),
    oracle parity, and a roofline whose `frac` recomputes from the declared
    work per launch and the measured launch time."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--e2e-reps", "2"],
                         capture_output=True, text=True, cwd=ROOT, timeout=1200)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert key in d, key
    assert d["config"]["workload"] == "c4" and d["n_gpus"] == 1
    assert d["config"]["n"] == 1 << 20 and d["config"]["m"] == 16384
    assert d["parity_vs_oracle"] is True
    assert d["gpu_launches"] > 0
    evals = d["config"]["n"] * d["config"]["m"] * d["config"]["afd_steps"]
    assert abs(d["value"] - evals / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    assert 0.3 * d["value"] < d["e2e"]["value"] < 1.05 * d["value"]
    r = d["roofline"]
    # the binding roofline of the (pruned) fast field: FP64 when most rows
    # run on chip, HBM when they take the two-pass path
    if r["bound"] == "hbm":
        assert r["unit"] == "GB/s"
        achieved = r["evals_per_launch"] * r["bytes_per_eval"] / (r["launch_ms"] * 1e-3) / 1e9
    else:
        assert r["bound"] == "fp64" and r["unit"] == "TFLOP/s"
        achieved = r["evals_per_launch"] * r["flops_per_eval"] / (r["launch_ms"] * 1e-3) / 1e12
    assert abs(achieved - r["achieved"]) <= 1e-6 * achieved
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 and 0.0 < r["frac"] < 1.0
    sp = r.get("split")
    if sp is not None:
        rows = d["config"]["m"]
        tiers = (32, 64, 128, 256, 512, 1024, 4096)
        assert sum(sp["rows_%d" % t] for t in tiers) == sp["onchip_rows"]
        assert sp["onchip_rows"] + sp["twopass_rows"] == rows
        assert all(sp["flops_per_eval_%d" % t] == 5 * (t.bit_length() - 1) + 7 for t in tiers)
        f = (sum(sp["rows_%d" % t] * sp["flops_per_eval_%d" % t] for t in tiers) +
             sp["twopass_rows"] * sp["flops_per_eval_twopass"]) / rows
        assert abs(f - r["flops_per_eval"]) <= 1e-9 * f
        assert abs(r["bytes_per_eval"] - 32.0 * sp["twopass_rows"] / rows) <= 1e-12
    assert r["evals_per_launch"] == d["config"]["n"] * d["config"]["m"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


# ---------------------------------------------------------------------------
# fast mode (AFD_PLAN_FAST / engine "fft-fast"): FMA-fused butterflies and
# on-chip r^l.  Contract (BASELINE north_star): identical selected indices,
# coefficients / remainders / errors within 1e-9 relative.  The field itself
# is checked much tighter (1e-12 of the row's largest value).
# ---------------------------------------------------------------------------
FAST_TOL = 1e-9


@pytest.mark.parametrize("n", [8, 16, 64, 256, 1024, 4096, 8192])
def test_fast_field_rows_close_to_reference(afd, tr, n):
    core, engine = afd
    import torch
    c = tr["fwd_%d" % n]
    radii = tuple(tr["radii_%d" % n])
    ref = tr["field_%d" % n]
    plan = engine.Plan(radii, n, fast=1)
    got = plan.field(torch.from_numpy(c).cuda()).cpu().numpy()
    for row in range(len(radii)):
        scale = np.abs(ref[row]).max()
        assert np.abs(got[row] - ref[row]).max() <= 1e-12 * scale, (n, row)


# Not the tie-prone cases: "atom" (after the exact one-atom recovery the
# residual is rounding noise, ~1e-31, and the next selection is decided by
# that noise) and the paper's f1/f2 signals (real Taylor coefficients: the
# field is conjugate-symmetric, so j and N - j tie up to the last bits and
# only the bit-exact engine reproduces the reference's pick).
@pytest.mark.parametrize("case", ["c0", "c1", "c3_s0", "c3_s1", "rand3", "rand11", "rand42",
                                  "const"])
def test_fast_decompose_matches_reference(afd, case):
    core, _ = afd
    g = load_golden("decomp_%s.npz" % case)
    thr = float(g["threshold"])
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    d = core.decompose(g["g"], grid, max_terms=int(g["max_terms"]),
                       threshold=None if np.isnan(thr) else thr,
                       dc_first=bool(g["dc_first"]), engine="fft-fast")
    assert d.engine == "fft-fast"
    assert len(d.steps) == len(g["j"])
    for k, s in enumerate(d.steps):
        assert s.point.angle_index == g["j"][k], (case, k)
        assert s.point.radius == g["radius"][k], (case, k)
        assert abs(s.coefficient - g["coeff"][k]) <= FAST_TOL * abs(g["coeff"][k]), (case, k)
        assert abs(s.residual_energy - g["residual"][k]) <= FAST_TOL * max(
            abs(g["residual"][k]), 1e-300 + FAST_TOL * g["initial"]), (case, k)
    scale = np.abs(g["remainder"]).max() + 1e-300
    assert np.abs(d.remainder - g["remainder"]).max() <= FAST_TOL * scale


def test_fast_c3_batch_matches_oracle(afd):
    """Batched fast decompositions (c3 shape, 8 signals): identical selections."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c3"]
    sig = np.stack([W.signal_for("c3", i) for i in range(8)])
    radii = W.radii_for(w.m)
    grid = core.ParameterGrid(radii, w.n)
    ds = core.decompose_batch(sig, grid, max_terms=w.steps, engine="fft-fast")
    for i in (0, 5):
        o = O.decompose(sig[i], np.array(radii), max_terms=w.steps)
        assert [s.point.angle_index for s in ds[i].steps] == list(o.steps["j"])
        assert [s.point.radius for s in ds[i].steps] == list(o.steps["radius"])
        c = np.array([s.coefficient for s in ds[i].steps])
        oc = o.steps["c_re"] + 1j * o.steps["c_im"]
        assert np.all(np.abs(c - oc) <= FAST_TOL * np.abs(oc))


@pytest.mark.parametrize("k,m", [(16, 100), (20, 5)])
def test_fast_big_field_rows_close_to_oracle(afd, k, m):
    """Fast large-N field (pass A with on-chip weights + (c, t) column pass):
    materialised rows vs the oracle's bit-exact rows, 1e-12 of each row's max."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 32, 0.98, 50 + k)
    radii = tuple(0.999 * i / (m - 1) for i in range(m))
    ghat = O.dft_forward(g)
    plan = engine.Plan(radii, n, fast=1)
    rows = [0, 1, m // 2, m - 1] if m > 4 else list(range(m))
    got = plan.field(torch.from_numpy(ghat).cuda()).cpu().numpy()
    for r in rows:
        ref = O.field(ghat, np.array(radii), r, r + 1)[0]
        assert np.abs(got[r] - ref).max() <= 1e-12 * np.abs(ref).max(), r


@pytest.mark.parametrize("k,m", [(16, 163), (20, 7)])
def test_fast_big_decompose_matches_oracle(afd, k, m):
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 32, 0.97, 7 + k)
    radii = tuple(i / m for i in range(m))
    d = core.decompose(g, core.ParameterGrid(radii, n), max_terms=3, engine="fft-fast")
    o = O.decompose(g, np.array(radii), max_terms=3)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    oc = o.steps["c_re"] + 1j * o.steps["c_im"]
    c = np.array([s.coefficient for s in d.steps])
    assert np.all(np.abs(c - oc) <= FAST_TOL * np.abs(oc))
    res = np.array([s.residual_energy for s in d.steps])
    assert np.all(np.abs(res - o.steps["residual"]) <= FAST_TOL * o.steps["residual"])
    assert np.abs(d.remainder - o.remainder).max() <= FAST_TOL * np.abs(o.remainder).max()


def test_fast_c2_first_steps(afd):
    """BASELINE c2 (N=65536, M=4096) in fast mode: the reference's own first
    selections (golden fixture) with coefficients / residuals within 1e-9."""
    core, _ = afd
    g = load_golden("c2_step.npz")
    grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
    d = core.decompose(g["g"], grid, max_terms=len(g["s"]), engine="fft-fast")
    for k, st in enumerate(d.steps):
        assert grid.radii.index(st.point.radius) == g["s"][k]
        assert st.point.angle_index == g["j"][k]
        assert abs(st.coefficient - g["coeff"][k]) <= FAST_TOL * abs(g["coeff"][k])
        assert abs(st.residual_energy - g["residual"][k]) <= FAST_TOL * g["residual"][k]


def test_fast_c4_full_size_replay(afd):
    """BASELINE c4 at full size (N = 2^20, M = 16384) in fast mode, 3 AFD
    steps, replayed by the oracle (selected row's first maximum, neighbouring
    and sampled rows, coefficient and residual within 1e-9 per step)."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c4"]
    g = W.signal_for("c4")
    radii = np.array(W.radii_for(w.m))
    plan = engine.Plan(tuple(radii), w.n, max_batch=1, fast=1)
    try:
        rec, counts, initial, rem, _, _ = plan.decompose_host(g[None, :], 3)
    finally:
        del plan
    r = O.replay_check(g, radii, rec[0], int(counts[0]), rows_per_step=4, rtol=FAST_TOL,
                       threads=O.max_threads())
    assert r["ok"], r["why"]
    assert np.abs(rem[0] - r["remainder"]).max() <= FAST_TOL * np.abs(r["remainder"]).max()


def test_c4_fast_and_exact_select_identically(afd):
    """BASELINE c4 at full size, all 20 AFD steps in both modes: the fast
    field selects exactly the exact (bit-identical to the reference) engine's
    grid points, with coefficients and residuals within 1e-9."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c4"]
    g = W.signal_for("c4")[None, :]
    radii = W.radii_for(w.m)
    p = engine.Plan(radii, w.n, max_batch=1, fast=1)
    rf, cf, _, remf, _, _ = p.decompose_host(g, w.steps)
    del p
    p = engine.Plan(radii, w.n, max_batch=1)
    re_, ce, _, reme, _, _ = p.decompose_host(g, w.steps)
    del p
    assert int(cf[0]) == int(ce[0]) == w.steps
    assert np.array_equal(rf[0]["s"], re_[0]["s"]) and np.array_equal(rf[0]["j"], re_[0]["j"])
    c1 = rf[0]["c_re"] + 1j * rf[0]["c_im"]
    c2 = re_[0]["c_re"] + 1j * re_[0]["c_im"]
    assert np.all(np.abs(c1 - c2) <= FAST_TOL * np.abs(c2))
    assert np.all(np.abs(rf[0]["residual"] - re_[0]["residual"]) <= FAST_TOL * re_[0]["residual"])
    assert np.all(re_[0]["flags"] == 0)  # every kernel norm from the libm pow table


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_c2_all_steps_replayed_by_oracle(afd, mode):
    """BASELINE c2 in full (N = 2^16, M = 4096, 50 AFD steps, projected real
    input): every step replayed by the oracle (selected row's first maximum,
    neighbouring and sampled rows, coefficient and residual) — bitwise for
    the exact engine, 1e-9 for the fast one."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c2"]
    g = O.analytic_projection(W.signal_for("c2"))
    radii = np.array(W.radii_for(w.m))
    plan = engine.Plan(tuple(radii), w.n, max_batch=1, fast=int(mode == "fast"))
    rec, counts, _, rem, _, _ = plan.decompose_host(g[None, :], w.steps)
    del plan
    assert int(counts[0]) == w.steps
    tol = 0.0 if mode == "exact" else FAST_TOL
    r = O.replay_check(g, radii, rec[0], w.steps, rows_per_step=4, rtol=tol,
                       threads=O.max_threads())
    assert r["ok"], r["why"]
    if mode == "exact":
        assert np.array_equal(rem[0], r["remainder"])
        assert np.all(rec[0]["flags"] == 0)


def test_c4_exact_all_steps_replayed_by_oracle(afd):
    """BASELINE c4 in full, exact engine, all 20 AFD steps replayed bitwise."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS["c4"]
    g = W.signal_for("c4")
    radii = np.array(W.radii_for(w.m))
    plan = engine.Plan(tuple(radii), w.n, max_batch=1)
    rec, counts, _, rem, _, _ = plan.decompose_host(g[None, :], w.steps)
    del plan
    assert int(counts[0]) == w.steps
    r = O.replay_check(g, radii, rec[0], w.steps, rows_per_step=3, threads=O.max_threads())
    assert r["ok"], r["why"]
    assert np.array_equal(rem[0], r["remainder"])


# ---------------------------------------------------------------------------
# pruned fast field (csrc/afd_pruned.cuh): rows with a negligible weight tail
# as on-chip 4096-point transforms of pre-twiddled spectra, the rest through
# the two-pass path from the first failing row on (decided on the device)
# ---------------------------------------------------------------------------
def _first_unprunable(ghat, radii, L=4096):
    """numpy statement of prune_rows_kernel's test: first row whose tail bound
    T r^L / (1 - r) exceeds 2^-64 max_{l<L} r^l |G^_l| (log2 domain), with a
    band of +-1e-6 in the exponent for the device's rounding."""
    a = np.abs(ghat)
    lt = np.log2(a.max())
    lg = np.where(a[:L] > 0, np.log2(np.where(a[:L] > 0, a[:L], 1.0)), -np.inf)
    lo = hi = len(radii)
    for s, r in enumerate(radii):
        if r == 0.0:
            continue
        lr = np.log2(r)
        b = np.max(np.arange(L) * lr + lg)
        tail = lt + L * lr - np.log2(1.0 - r)
        if tail > b - 64.0 + 1e-6:
            hi = min(hi, s)
        if tail > b - 64.0 - 1e-6:
            lo = min(lo, s)
    return lo, hi


@pytest.mark.parametrize("radii", [
    tuple(i / 64 for i in range(64)),                                   # c2-like tail
    (0.3, 0.999, 0.5, 0.9, 0.99995, 0.1, 0.7, 0.0, 0.95, 0.2),          # unsorted, early long row
    (0.0, 0.2, 0.4),                                                    # all on chip
    (0.9999, 0.99999, 0.5),                                             # long rows first
])
def test_pruned_field_argmax_and_split(afd, radii):
    """The pruned field's first maximum is the oracle's (same flat index,
    |F|^2 within 1e-12), and the device's on-chip / two-pass split is the
    first row failing the tail test."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import workloads as W
    n = 1 << 16
    g = W.pole_sum(n, 32, 0.995, 99)
    ghat = O.dft_forward(g)
    plan = engine.Plan(radii, n, fast=1)
    got = np.frombuffer(plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes(),
                        O.CAND_DTYPE)[0]
    onchip, twopass = plan.field_split()
    n1k, n4k, n2p = plan.field_tiers()
    ref = O.field_argmax(ghat, np.array(radii))
    assert int(got["flat"]) == int(ref["flat"])
    assert abs(got["mag"] - ref["mag"]) <= 1e-12 * ref["mag"]
    lo, hi = _first_unprunable(ghat, radii)
    assert lo <= onchip <= hi and onchip + twopass == len(radii)
    lo1, hi1 = _first_unprunable(ghat, radii, L=1024)
    assert lo1 <= n1k <= hi1 and n1k + n4k == onchip and n2p == twopass
    # the register tiers (32, 64, 128 spectrum terms) inside the <= 1024 rows
    tr = plan.field_tier_rows()
    assert list(tr) == [32, 64, 128, 256, 512, 1024, 4096, n]
    assert sum(tr.values()) == len(radii) and tr[4096] == n4k and tr[n] == n2p
    assert sum(tr[L] for L in (32, 64, 128, 256, 512, 1024)) == n1k
    upto = 0
    for L in (32, 64, 128, 256, 512):
        lo_l, hi_l = _first_unprunable(ghat, radii, L=L)
        upto += tr[L]
        assert lo_l <= upto <= hi_l, L


# ---------------------------------------------------------------------------
# register tiers of the pruned field (csrc/afd_field_reg.cuh): rows that need
# at most 32, 64 or 128 spectrum terms, one thread per 32 outputs
# ---------------------------------------------------------------------------
def _cand(plan, ghat):
    import torch
    return np.frombuffer(plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes(),
                         O.CAND_DTYPE)[0]


@pytest.mark.parametrize("k", [16, 20])
def test_reg_tier_rows_one_by_one(afd, k):
    """Single-row fields at radii across the register and sub-warp tiers (and
    just beyond): each row's first maximum is the oracle's (flat index; value and
    magnitude to 1e-12), and the row went to the expected tier."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << k
    g = W.pole_sum(n, 24, 0.9, 4242 + k)
    ghat = O.dft_forward(g)
    rs = (0.0, 0.03, 0.11, 0.2, 0.249, 0.27, 0.33, 0.41, 0.499, 0.52, 0.61, 0.68, 0.73, 0.8,
          0.83, 0.86, 0.9, 0.93) if k == 16 else (0.17, 0.38, 0.6, 0.78, 0.89)
    for r in rs:
        plan = engine.Plan((r,), n, fast=1)
        got = _cand(plan, ghat)
        tr = plan.field_tier_rows()
        del plan
        ref = O.field_argmax(ghat, np.array([r]))
        assert int(got["flat"]) == int(ref["flat"]), r
        assert abs(got["mag"] - ref["mag"]) <= 1e-12 * ref["mag"], r
        assert abs(complex(got["re"], got["im"]) - complex(ref["re"], ref["im"])) \
            <= 1e-12 * np.sqrt(ref["mag"]), r
        want = next((L for L in (32, 64, 128, 256, 512)
                     if _first_unprunable(ghat, (r,), L=L)[0] == 1), 1024)
        assert tr[want] == 1, (r, tr)


def test_default_tier_choice(afd):
    """Without AFD_SUB_MIN_EVALS (the tests force the 256- / 512-point tiers
    on) a mid-size plan leaves their rows on the 1024-point tier, a c4-size
    radius grid uses them; the first maximum is the oracle's either way."""
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O
from paper_1711_08604_b200 import engine, workloads as W
out = {}
for name, n, m in (("mid", 1 << 16, 96), ("big", 1 << 20, 16384)):
    radii = tuple(0.97 * i / m for i in range(m))
    plan = engine.Plan(radii, n, fast=1)
    ghat = O.dft_forward(W.pole_sum(n, 12, 0.9, 31))
    got = np.frombuffer(plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes(),
                        O.CAND_DTYPE)[0]
    out[name] = {"tiers": [int(k) for k in plan.field_tier_rows()], "flat": int(got["flat"])}
    if name == "mid":
        out[name]["ref"] = int(O.field_argmax(ghat, np.array(radii))["flat"])
    del plan
print(json.dumps(out))
''' % ROOT
    env = {k: v for k, v in os.environ.items() if k != "AFD_SUB_MIN_EVALS"}
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["mid"]["tiers"] == [32, 64, 128, 1024, 4096, 1 << 16]
    assert out["mid"]["flat"] == out["mid"]["ref"]
    assert out["big"]["tiers"] == [32, 64, 128, 256, 512, 1024, 4096, 1 << 20]


@pytest.mark.parametrize("engine_name", ["fft-fast", "fft-fast-margins"])
def test_reg_tier_low_radius_grid_decomposes_like_the_oracle(afd, engine_name):
    """Every radius <= 0.69: the whole field runs in the register tiers, so
    every selection comes from them (many rows per CTA, several CTAs per
    row block, descending row order): identical poles, 1e-9 values, and the
    reference's margins."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n, m = 1 << 16, 300
    radii = tuple(0.69 * i / (m - 1) for i in range(m))
    g = W.pole_sum(n, 16, 0.75, 777)
    grid = core.ParameterGrid(radii, n)
    d = core.decompose(g, grid, max_terms=4, engine=engine_name)
    o = O.decompose(g, np.array(radii), max_terms=4)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    oc = o.steps["c_re"] + 1j * o.steps["c_im"]
    c = np.array([s.coefficient for s in d.steps])
    assert np.all(np.abs(c - oc) <= FAST_TOL * np.abs(oc))
    assert np.abs(d.remainder - o.remainder).max() <= FAST_TOL * np.abs(o.remainder).max()
    if engine_name.endswith("margins"):
        ref = _oracle_margins(g, radii, o.steps)
        assert np.all(np.abs(np.array(d.margins) - ref) <= 1e-9)


def test_reg_tier_ties_take_the_lowest_flat_index(afd):
    """Exact ties inside the register tiers: a constant signal (every point
    of a row equal, the r = 0 row the largest) and duplicated radii (equal
    rows): the first maximum in flat order wins although rows are visited in
    decreasing order and every thread holds an equal candidate."""
    core, engine = afd
    n = 1 << 16
    ghat = O.dft_forward(np.full(n, 0.75 - 0.25j))
    plan = engine.Plan((0.0, 0.1, 0.2), n, fast=1)
    got = _cand(plan, ghat)
    assert plan.field_tier_rows()[32] == 3
    del plan
    assert int(got["flat"]) == 0 == int(O.field_argmax(ghat, np.array([0.0, 0.1, 0.2]))["flat"])
    from paper_1711_08604_b200 import workloads as W
    ghat = O.dft_forward(W.pole_sum(n, 8, 0.8, 5))
    radii = (0.1, 0.3, 0.2, 0.3, 0.3, 0.05)
    plan = engine.Plan(radii, n, fast=1)
    got = _cand(plan, ghat)
    del plan
    ref = O.field_argmax(ghat, np.array(radii))
    assert int(got["flat"]) == int(ref["flat"])
    assert int(ref["flat"]) // n == 1


def test_pruned_fast_decompose_long_rows_and_threshold(afd):
    """A fast decomposition whose grid mixes on-chip and two-pass rows (radii
    up to 0.99999) and stops on the threshold: identical poles and 1e-9
    against the oracle, and the same number of steps."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n = 1 << 16
    radii = (0.0, 0.2, 0.5, 0.8, 0.9, 0.97, 0.999, 0.99999)
    g = W.pole_sum(n, 8, 0.999, 123)
    grid = core.ParameterGrid(radii, n)
    d = core.decompose(g, grid, max_terms=12, threshold=0.02, engine="fft-fast")
    o = O.decompose(g, np.array(radii), max_terms=12, threshold=0.02)
    assert len(d.steps) == len(o.steps)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    assert [s.point.radius for s in d.steps] == list(o.steps["radius"])
    oc = o.steps["c_re"] + 1j * o.steps["c_im"]
    c = np.array([s.coefficient for s in d.steps])
    assert np.all(np.abs(c - oc) <= FAST_TOL * np.abs(oc))
    assert np.abs(d.remainder - o.remainder).max() <= FAST_TOL * np.abs(o.remainder).max()


# ---------------------------------------------------------------------------
# register tiers for batches of on-chip fields (pruned_small in afd_capi.cu,
# BASELINE c3's regime): per-signal tier limits, hints and candidate rows
# ---------------------------------------------------------------------------
def _batch_cands(plan, ghat):
    import torch
    raw = plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes()
    return np.frombuffer(raw, O.CAND_DTYPE)


@pytest.mark.parametrize("n,m,b", [(4096, 1024, 64), (1024, 1024, 256), (8192, 512, 64),
                                   (2048, 512, 256), (1024, 1024, 260), (4096, 1000, 67)])
def test_small_pruned_batch_field_argmax(afd, n, m, b):
    """A batch large enough for the register tiers (batch x rows x N >= 2^28):
    every signal's first maximum is the oracle's — signals whose poles sit at
    small radii (maximum inside a register tier), at large radii (N-point
    rows), a constant (exact ties, flat index 0) — and the tier rows add up."""
    core, engine = afd
    from paper_1711_08604_b200 import workloads as W
    radii = tuple(i / m for i in range(m))
    rmax = (0.2, 0.45, 0.65, 0.9, 0.97)
    sig = np.stack([W.pole_sum(n, 6, rmax[i % 5], 9000 + i) for i in range(b)])
    sig[3] = 0.5 - 0.125j
    ghat = np.stack([O.dft_forward(x) for x in sig])
    plan = engine.Plan(radii, n, max_batch=b, fast=1)
    got = _batch_cands(plan, ghat)
    tr = plan.field_tier_rows()
    del plan
    # N >= 4096: rows that need up to 1024 terms run as N / 1024 warp-per-row fields
    # (ragged batches: the last CTAs of the register kernels are partly idle)
    assert list(tr) == ([32, 64, 128, 256, 512, 1024, n] if n >= 4096 else [32, 64, 128, n])
    assert sum(tr.values()) == b * m and all(v > 0 for v in tr.values())
    tiers_hit = set()
    for i in list(range(0, b, 7)) + [3]:
        ref = O.field_argmax(ghat[i], np.array(radii), threads=O.max_threads())
        assert int(got[i]["flat"]) == int(ref["flat"]), i
        assert abs(got[i]["mag"] - ref["mag"]) <= 1e-12 * ref["mag"], i
        tiers_hit.add(min(3, int(radii[int(ref["flat"]) // n] * 4)))
    assert int(got[3]["flat"]) == 0
    assert len(tiers_hit) >= 2


@pytest.mark.parametrize("engine_name", ["fft-fast", "fft-fast-margins"])
def test_small_pruned_batch_decompose(afd, engine_name):
    """decompose_batch through the register tiers (64 signals of N = 4096 on
    1024 radii), some signals stopping on the threshold: identical poles,
    1e-9 values and the reference's margins for a sample of the signals."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n, m, b, steps = 4096, 1024, 64, 4
    radii = tuple(i / m for i in range(m))
    rmax = (0.3, 0.6, 0.95)
    sig = np.stack([W.pole_sum(n, 2 if i % 4 == 1 else 12, rmax[i % 3], 500 + i)
                    for i in range(b)])
    grid = core.ParameterGrid(radii, n)
    ds = core.decompose_batch(sig, grid, max_terms=steps, threshold=1e-3, engine=engine_name)
    stopped = 0
    for i in (0, 1, 2, 5, 13, 30, 63):
        o = O.decompose(sig[i], np.array(radii), max_terms=steps, threshold=1e-3)
        stopped += len(o.steps) < steps
        assert len(ds[i].steps) == len(o.steps), i
        assert [s.point.angle_index for s in ds[i].steps] == list(o.steps["j"]), i
        assert [s.point.radius for s in ds[i].steps] == list(o.steps["radius"]), i
        c = np.array([s.coefficient for s in ds[i].steps])
        oc = o.steps["c_re"] + 1j * o.steps["c_im"]
        assert np.all(np.abs(c - oc) <= FAST_TOL * np.abs(oc)), i
        scale = np.abs(o.remainder).max() + 1e-300
        assert np.abs(ds[i].remainder - o.remainder).max() <= FAST_TOL * scale, i
        if engine_name.endswith("margins") and i in (0, 2):
            ref = _oracle_margins(sig[i], radii, o.steps)
            assert np.all(np.abs(np.array(ds[i].margins) - ref) <= 1e-9), i
    assert stopped >= 1


# ---------------------------------------------------------------------------
# per-step top-2 margins (fast engine)
# ---------------------------------------------------------------------------
def _oracle_margins(g, radii, steps):
    """The reference's own top-2 relative margin of |F|^2 at every step:
    replay the oracle's selections, full field each step."""
    out = []
    rem = np.ascontiguousarray(g, dtype=np.complex128)
    for rec in steps:
        f = O.field(O.dft_forward(rem), np.array(radii))
        mag = (f.real * f.real + f.imag * f.imag).ravel()
        top = np.argmax(mag)
        best = mag[top]
        mag[top] = -1.0
        out.append((best - max(mag.max(), 0.0)) / best)
        rem = O.remainder_update(rem, complex(rec["a_re"], rec["a_im"]),
                                 complex(rec["c_re"], rec["c_im"]))
    return np.array(out)


@pytest.mark.parametrize("n,m,poles,steps", [(1024, 100, 8, 10), (4096, 96, 16, 6),
                                             (1 << 16, 12, 16, 3)])
def test_fast_margins_match_the_reference(afd, n, m, poles, steps):
    """engine "fft-fast-margins" reports each step's top-2 relative margin;
    it is the reference's (full-field replay) to 1e-9 absolute (on-chip N,
    the cluster and one-CTA step kernels, and the pruned + two-pass large-N
    field).  Exact and plain fast decompositions report NaN."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    g = W.pole_sum(n, poles, 0.99 if n > 8192 else 0.95, 1000 + n)
    radii = tuple(0.9995 * i / (m - 1) for i in range(m)) if n > 8192 else \
        tuple(i / m for i in range(m))
    grid = core.ParameterGrid(radii, n)
    d = core.decompose(g, grid, max_terms=steps, engine="fft-fast-margins")
    o = O.decompose(g, np.array(radii), max_terms=steps)
    assert [s.point.angle_index for s in d.steps] == list(o.steps["j"])
    ref = _oracle_margins(g, radii, o.steps)
    got = np.array(d.margins)
    assert got.shape == ref.shape and np.all(np.isfinite(got))
    assert np.all(np.abs(got - ref) <= 1e-9), (got, ref)
    # the same selections as the margin-free fast engine; exact and plain
    # fast decompositions report NaN
    f = core.decompose(g, grid, max_terms=steps, engine="fft-fast")
    assert [s.point.angle_index for s in f.steps] == [s.point.angle_index for s in d.steps]
    assert all(np.isnan(x) for x in f.margins)
    e = core.decompose(g, grid, max_terms=2, engine="fft")
    assert len(e.margins) == 2 and all(np.isnan(x) for x in e.margins)


def test_fast_batch_margins(afd):
    """decompose_batch with margins: every signal's margins as its own."""
    core, _ = afd
    from paper_1711_08604_b200 import workloads as W
    n, m = 4096, 64
    radii = tuple(i / m for i in range(m))
    sig = np.stack([W.pole_sum(n, 16, 0.95, 70 + s) for s in range(3)])
    grid = core.ParameterGrid(radii, n)
    ds = core.decompose_batch(sig, grid, max_terms=4, engine="fft-fast-margins")
    for i in range(3):
        o = O.decompose(sig[i], np.array(radii), max_terms=4)
        ref = _oracle_margins(sig[i], radii, o.steps)
        assert np.all(np.abs(np.array(ds[i].margins) - ref) <= 1e-9)


@pytest.mark.parametrize("n", [1024, 2048, 4096])
@pytest.mark.parametrize("fast", [0, 1])
def test_tmem_field_variants_full_groups(afd, n, fast):
    """The TMEM field kernel at N = 1024 (eight row-groups of 64 threads: two
    groups fill the four lane quadrants), 2048 (four groups) and 4096 (two),
    launched with every group busy: materialised rows bitwise (exact) or to
    1e-12 of the row's largest value (fast) against the oracle, and the
    first maximum."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import workloads as W
    m = 512
    radii = tuple(0.99 * i / m for i in range(m))
    g = W.pole_sum(n, 16, 0.95, 7 + n)
    ghat = O.dft_forward(g)
    plan = engine.Plan(radii, n, fast=fast)
    got = plan.field(torch.from_numpy(ghat).cuda()).cpu().numpy()
    ref = O.field(ghat, np.array(radii))
    if fast:
        scale = np.abs(ref).max(axis=1, keepdims=True)
        assert np.all(np.abs(got - ref) <= 1e-12 * scale)
    else:
        assert np.array_equal(got, ref)
    c = np.frombuffer(plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes(),
                      O.CAND_DTYPE)[0]
    r = O.field_argmax(ghat, np.array(radii))
    assert int(c["flat"]) == int(r["flat"])


@pytest.mark.parametrize("fast", [0, 1])
def test_field_n512_many_signals(afd, fast):
    """N = 512 with enough signals that every CTA runs all sixteen one-warp
    row-groups (a regression: named barriers 1..16 overflowed the 16 a CTA
    has); argmax per signal against the oracle."""
    core, engine = afd
    import torch
    from paper_1711_08604_b200 import workloads as W
    n, m, b = 512, 256, 32
    radii = tuple(i / m for i in range(m))
    sig = np.stack([W.pole_sum(n, 8, 0.95, 300 + i) for i in range(b)])
    ghat = np.stack([O.dft_forward(x) for x in sig])
    plan = engine.Plan(radii, n, max_batch=b, fast=fast)
    got = np.frombuffer(plan.field_argmax(torch.from_numpy(ghat).cuda()).cpu().numpy().tobytes(),
                        O.CAND_DTYPE)
    for i in range(b):
        r = O.field_argmax(ghat[i], np.array(radii))
        assert int(got[i]["flat"]) == int(r["flat"]), i
        if not fast:
            assert got[i]["mag"] == r["mag"]
