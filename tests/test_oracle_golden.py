"""Pin the CPU oracle (oracle/afd_oracle.c) against the reference's own outputs.

The fixtures were produced by running /root/reference (tests/golden/
make_golden.py); equality here is exact (np.array_equal, i.e. bitwise up to
the sign of zero), which is what licenses the oracle as the parity checker
for the CUDA path.
"""

import numpy as np
import pytest

import oracle as O
from conftest import DECOMP_CASES, load_golden


@pytest.fixture(scope="module")
def tr():
    return load_golden("transforms.npz")


@pytest.mark.parametrize("n", [8, 16, 64, 256, 1024, 4096, 8192])
def test_transforms_bitwise(tr, n):
    x = tr["x_%d" % n]
    assert np.array_equal(O.dft_forward(x), tr["fwd_%d" % n])
    assert np.array_equal(O.dft_inverse(x), tr["inv_%d" % n])
    c = tr["fwd_%d" % n]
    assert np.array_equal(O.field(c, tr["radii_%d" % n]), tr["field_%d" % n])
    assert O.energy(x) == tr["energy_%d" % n]
    assert O.cmean(x) == tr["mean_%d" % n]
    assert np.array_equal(O.analytic_projection(tr["xr_%d" % n]), tr["proj_%d" % n])
    a, c2 = complex(tr["a_%d" % n]), complex(tr["c_%d" % n])
    assert np.array_equal(O.kernel_samples(a, n), tr["ks_%d" % n])
    assert np.array_equal(O.blaschke_samples(a, n), tr["bs_%d" % n])
    assert np.array_equal(O.remainder_update(x, a, c2), tr["upd_%d" % n])


@pytest.mark.parametrize("case", DECOMP_CASES)
def test_decompose_bitwise(case):
    g = load_golden("decomp_%s.npz" % case)
    thr = float(g["threshold"])
    d = O.decompose(g["g"], g["radii"], max_terms=int(g["max_terms"]),
                    threshold=None if np.isnan(thr) else thr, dc_first=bool(g["dc_first"]))
    st = d.steps
    assert len(st) == len(g["j"])
    assert np.array_equal(st["j"], g["j"])
    assert np.array_equal(st["radius"], g["radius"])
    assert np.array_equal(st["a_re"] + 1j * st["a_im"], g["a"])
    assert np.array_equal(st["c_re"] + 1j * st["c_im"], g["coeff"])
    assert np.array_equal(st["residual"], g["residual"])
    assert d.initial_energy == g["initial"]
    assert np.array_equal(d.remainder, g["remainder"])
    if len(st):
        errs, total = O.error_trace(g["g"], st)
        assert np.array_equal(errs, g["trace"])
        assert np.array_equal(total, g["reconstruction"])


def test_c2_first_steps():
    """BASELINE c2 (N=65536, M=4096, real input): projection + 2 selections."""
    g = load_golden("c2_step.npz")
    proj = O.analytic_projection(g["x"])
    assert np.array_equal(proj, g["g"])
    rem = proj
    radii = g["radii"]
    z = O.circle(rem.shape[0])
    for k in range(len(g["s"])):
        best = O.field_argmax(O.dft_forward(rem), radii)
        s, j = divmod(int(best["flat"]), rem.shape[0])
        assert (s, j) == (int(g["s"][k]), int(g["j"][k]))
        coeff = complex(best["re"], best["im"])
        assert coeff == g["coeff"][k]
        a = complex(radii[s] * z[j].real, radii[s] * z[j].imag)
        rem = O.remainder_update(rem, a, coeff)
        assert O.energy(rem) == g["residual"][k]
    assert np.array_equal(rem, g["remainder"])


def test_workload_generators_stable():
    """The seeded BASELINE inputs regenerate bit-identically (fixtures hold them)."""
    from paper_1711_08604_b200 import workloads as W
    assert np.array_equal(W.signal_for("c0"), load_golden("decomp_c0.npz")["g"])
    assert np.array_equal(W.signal_for("c3", 1), load_golden("decomp_c3_s1.npz")["g"])
    assert np.array_equal(W.signal_for("c2"), load_golden("c2_step.npz")["x"])


def _big_input(n, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


@pytest.mark.parametrize("n", [16384, 65536, 1 << 20])
def test_big_n_elision_forms(n):
    """N >= 16384: numpy's temporary elision swaps multiply operands."""
    b = load_golden("big.npz")
    x = _big_input(n, n)
    sel = np.arange(0, n, 4099) if n > 16384 else np.arange(n)
    a, c = complex(b["a_%d" % n]), complex(b["c_%d" % n])
    assert np.array_equal(O.dft_forward(x)[sel], b["fwd_%d" % n])
    assert np.array_equal(O.dft_inverse(x)[sel], b["inv_%d" % n])
    assert np.array_equal(O.kernel_samples(a, n)[sel], b["ks_%d" % n])
    assert np.array_equal(O.blaschke_samples(a, n)[sel], b["bs_%d" % n])
    upd = O.remainder_update(x, a, c)
    assert np.array_equal(upd[sel], b["upd_%d" % n])
    assert O.energy(x) == b["energy_%d" % n]
    assert O.energy(upd) == b["upd_energy_%d" % n]
    assert O.cmean(x) == b["mean_%d" % n]
    if n <= 65536:
        f = O.field(O.dft_forward(x), b["radii_%d" % n])
        assert np.array_equal(f[:, sel], b["field_%d" % n])


def test_numpy_port_field_matches_the_c_oracle():
    """oracle/numpy_port.py (the reference's numpy selection step, timed by
    bench.py as the reference-speed baseline) computes the C oracle's field
    bit for bit and the same first maximum."""
    import oracle as O
    from oracle import numpy_port as NP
    from paper_1711_08604_b200 import workloads as W
    for n, m, seed in ((1024, 100, 3), (4096, 64, 4), (1 << 14, 8, 5)):
        g = W.pole_sum(n, 16, 0.95, seed)
        radii = W.radii_for(m)
        c = O.dft_forward(g)
        t = NP.Tables(radii, n)
        assert np.array_equal(NP.field(t, c), O.field(c, np.array(radii)))
        s, j, mag, f = NP.select(t, c)
        cand = O.field_argmax(c, np.array(radii))
        assert (s * n + j, mag) == (int(cand["flat"]), float(cand["mag"]))
