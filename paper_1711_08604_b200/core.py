"""Reference-compatible AFD API, computed on the B200.

Mirrors ``fastafd.core`` (``/root/reference/pkg/src/fastafd/core.py``):
same names, signatures, argument meaning, return types and ``ValueError``
behaviour, so code written against the reference switches by changing the
import.  Host-side work is limited to argument validation, building the
reference's plain-data result objects and copying arrays across PCIe; every
number is produced by a kernel of ``libafd_b200.so`` through the C ABI
(``include/afd_capi.h``), bit-identical to the reference's numpy arithmetic
(see ``csrc/afd_common.cuh``).  There is no CPU fallback: without a CUDA
device or the built library every compute entry point raises
``AfdCudaUnavailable``.

Engines.  ``engine="fft"`` is the reference's transform engine (the hot
path accelerated here), bit-identical to the reference.  ``engine="direct"``
is the reference's O(M N^2) quadrature baseline (``oracle.field_direct``),
also on the device (``csrc/afd_direct.cuh``, N <= 8192); its sums are
ordered differently from np.correlate, so it agrees with the reference to
the reference's own engine tolerance (identical poles, 1e-9), not bitwise.
``engine="fft-fast"`` (an addition; the reference has no such engine) is
the transform engine with the field computed in fast FP64 arithmetic
(AFD_PLAN_FAST: FMA-fused butterflies, r^l formed on chip): the selected
poles are identical to the reference's and coefficients, remainders and
errors agree to ~1e-14 relative (the north-star contract is 1e-9).
``engine="fft-fast-margins"`` is the same engine with each step's top-2
relative margin of |F|^2 over the grid recorded in ``Decomposition.margins``
(~10-15% slower field).
``parallel`` is accepted for signature compatibility; the device path is
always parallel and, like the reference's threaded path, produces
identical results.
"""

from __future__ import annotations

import gc
import warnings
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _capi

__all__ = [
    "radius_range", "ParameterPoint", "ParameterGrid", "DecompositionStep", "Decomposition",
    "discrete_energy", "analytic_projection", "kernel_samples", "blaschke_samples",
    "spectral_coefficients", "inner_product_field", "maximal_selection", "remainder_update",
    "decompose", "decompose_batch", "tm_basis_samples", "reconstruct", "relative_error",
    "error_trace", "ENGINES",
]

RADIUS_WARN_LIMIT = 0.95  # core.py:59
ENGINES = ("fft", "direct", "fft-fast", "fft-fast-margins")
_FAST_LEVEL = {"fft-fast": 1, "fft-fast-margins": 2}  # engine.Plan(fast=...)


def _engine():
    from . import engine  # imports torch; deferred so validation works without it
    return engine


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# grids and validation (core.py:62-167)
# ---------------------------------------------------------------------------

def radius_range(start, step, stop):
    """start, start+step, ... up to and including stop, with 1e-9 slack (core.py:62-69)."""
    if step <= 0:
        raise ValueError("step must be positive")
    count = int(np.floor((stop - start) / step + 1e-9)) + 1
    if count < 1:
        raise ValueError("empty radius range")
    return tuple(start + k * step for k in range(count))


def _is_pow2(n, low):
    return n >= low and (n & (n - 1)) == 0


def _as_signal(x):
    """Validated complex128 1-d power-of-two signal (core.py:72-81)."""
    g = np.asarray(x, dtype=np.complex128)
    if g.ndim != 1:
        raise ValueError("signal must be 1-d, got shape %r" % (g.shape,))
    if not _is_pow2(g.shape[0], 8):
        raise ValueError("signal length must be a power of two >= 8, got %d" % g.shape[0])
    if not np.all(np.isfinite(g)):
        raise ValueError("signal contains non-finite samples")
    return g


def _pole_value(a):
    v = complex(a.value) if isinstance(a, ParameterPoint) else complex(a)
    if abs(v) >= 1.0:
        raise ValueError("pole must lie strictly inside the unit disc, got |a|=%g" % abs(v))
    return v


@dataclass(frozen=True)
class ParameterPoint:
    """Candidate pole a = r exp(2 pi i j / N) (core.py:100-112)."""

    radius: float
    angle_index: int
    value: complex

    def __post_init__(self):
        if not 0.0 <= self.radius < 1.0:
            raise ValueError("radius must satisfy 0 <= r < 1, got %g" % self.radius)
        if abs(self.value) >= 1.0:
            raise ValueError("pole modulus must be < 1")


@dataclass(frozen=True)
class ParameterGrid:
    """M radii times N angles (core.py:115-167)."""

    radii: tuple
    angular_count: int

    def __post_init__(self):
        radii = tuple(float(r) for r in self.radii)
        object.__setattr__(self, "radii", radii)
        if not radii:
            raise ValueError("grid needs at least one radius")
        bad = [r for r in radii if not 0.0 <= r < 1.0]
        if bad:
            raise ValueError("grid radii must lie in [0, 1), got %g" % bad[0])
        if any(hi <= lo for lo, hi in zip(radii, radii[1:])):
            raise ValueError("grid radii must be strictly increasing")
        if not _is_pow2(self.angular_count, 8):
            raise ValueError("angular_count must be a power of two >= 8, got %d"
                             % self.angular_count)
        if radii[-1] > RADIUS_WARN_LIMIT:
            warnings.warn("largest grid radius %g exceeds %g; the 1/(1-r^N) weighting "
                          "degrades close to the unit circle" % (radii[-1], RADIUS_WARN_LIMIT),
                          stacklevel=2)

    @classmethod
    def from_range(cls, start, step, stop, angular_count):
        return cls(radius_range(start, step, stop), angular_count)

    @classmethod
    def evenly_spaced(cls, count, angular_count):
        return cls(tuple(s / (count + 1) for s in range(1, count + 1)), angular_count)

    @classmethod
    def experiment_default(cls, angular_count):
        return cls.from_range(0.0, 0.1, 0.8, angular_count)

    def point(self, radius_index, angle_index):
        r = self.radii[radius_index]
        value = r * np.exp(2j * np.pi * angle_index / self.angular_count)
        return ParameterPoint(r, int(angle_index), complex(value))


@dataclass(frozen=True)
class DecompositionStep:
    point: ParameterPoint
    coefficient: complex
    residual_energy: float


@dataclass(eq=False)
class Decomposition:
    steps: tuple
    grid: ParameterGrid
    n_samples: int
    initial_energy: float
    engine: str
    remainder: np.ndarray | None = field(default=None, repr=False)
    # Per-step device flags (bit 0: CPython's pow(|a|, 2) not provably equal
    # to |a|*|a| for this pole, see csrc/afd_common.cuh).  Not in the reference.
    step_flags: tuple = field(default=(), repr=False)
    # Per-step top-2 relative margin of |F|^2 over the grid (fast engine;
    # NaN where not tracked), SURVEY.md §7.3(a).  Not in the reference.
    margins: tuple = field(default=(), repr=False)

    def poles(self):
        return np.array([s.point.value for s in self.steps], dtype=np.complex128)

    def __len__(self):
        return len(self.steps)


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

@lru_cache(maxsize=64)
def _circle_plan_radii(n):
    return (0.0,)


def _plan(n, radii=None, batch=1):
    return _engine().get_plan(_circle_plan_radii(n) if radii is None else radii, n, batch=batch)


def _to_dev(a, plan):
    t = _torch()
    return t.from_numpy(np.ascontiguousarray(a)).to(plan.device)


def _host(t):
    return t.cpu().numpy()


# ---------------------------------------------------------------------------
# energies, projection, atoms (core.py:195-245)
# ---------------------------------------------------------------------------

def discrete_energy(g):
    """(1/N) sum |G[m]|^2 (core.py:195-198)."""
    g = _as_signal(g)
    p = _plan(g.shape[0])
    return float(_host(p.energy(_to_dev(g, p)))[0])


def analytic_projection(x):
    """Real samples -> discrete analytic signal with the same real part (core.py:201-231)."""
    x = np.asarray(x)
    if np.iscomplexobj(x):
        if np.any(x.imag != 0):
            raise ValueError("analytic projection expects real input")
        x = x.real
    if not np.all(np.isfinite(x)):
        raise ValueError("input contains non-finite samples")
    if x.ndim != 1:
        raise ValueError("expected a 1-d buffer, got shape %r" % (x.shape,))
    n = x.shape[0]
    if n < 2 or n & (n - 1):
        raise ValueError("length must be a power of two >= 2, got %d" % n)
    if n < 8:
        raise ValueError("need at least 8 samples, got %d" % n)
    p = _plan(n)
    xc = np.asarray(x, dtype=np.float64).astype(np.complex128)
    return _host(p.analytic_projection(_to_dev(xc, p)))[0]


def _kernel_norm(value):
    """sqrt(1 - |a|^2) exactly as the reference evaluates it (core.py:237):
    CPython's abs (libm hypot) and float ** 2 (libm pow) on the host, so the
    device atoms use the reference's bits (afd_atom's `norm`)."""
    return float(np.sqrt(1.0 - abs(value) ** 2))


def kernel_samples(a, n):
    """sqrt(1-|a|^2)/(1 - conj(a) z) on the circle (core.py:234-238)."""
    v = _pole_value(a)
    p = _plan(int(n))
    return _host(p.atom(0, v, norm=_kernel_norm(v)))


def blaschke_samples(a, n):
    """(z - a)/(1 - conj(a) z) on the circle (core.py:241-245)."""
    v = _pole_value(a)
    p = _plan(int(n))
    return _host(p.atom(1, v))


def spectral_coefficients(g):
    """Forward-DFT coefficients of a validated signal (core.py:248-250)."""
    g = _as_signal(g)
    p = _plan(g.shape[0])
    return _host(p.dft_forward(_to_dev(g, p)))[0]


def inner_product_field(c, grid, parallel=False):
    """All grid inner products <G, e_a> as an (M, N) matrix (core.py:259-282)."""
    c = np.asarray(c, dtype=np.complex128)
    if c.ndim != 1 or c.shape[0] != grid.angular_count:
        raise ValueError("coefficient length %r does not match grid angular_count %d"
                         % (c.shape, grid.angular_count))
    p = _plan(grid.angular_count, grid.radii)
    return _host(p.field(_to_dev(c, p)))


def maximal_selection(field_values, grid):
    """Largest |<G, e_a>|^2, ties to the lowest (s, j) row-major (core.py:285-300)."""
    f = np.asarray(field_values)
    expected = (len(grid.radii), grid.angular_count)
    if f.shape != expected:
        raise ValueError("field shape %r does not match grid %r" % (f.shape, expected))
    if f.size == 0:
        raise ValueError("empty field")
    p = _plan(grid.angular_count, grid.radii)
    cand = _host(p.argmax(_to_dev(f.astype(np.complex128), p))).view(_capi.CAND_DTYPE)[0]
    s, j = divmod(int(cand["flat"]), grid.angular_count)
    return grid.point(s, j), complex(f[s, j])


def remainder_update(g, a, c):
    """(G - c e_a)(1 - conj(a) z)/(z - a) (core.py:303-314)."""
    g = _as_signal(g)
    v = _pole_value(a)
    p = _plan(g.shape[0])
    return _host(p.atom(2, v, complex(c), g=_to_dev(g, p), norm=_kernel_norm(v)))


# ---------------------------------------------------------------------------
# decompose (core.py:317-391)
# ---------------------------------------------------------------------------

def _check_decompose_args(g, grid, max_terms, threshold, engine):
    if grid.angular_count != g.shape[-1]:
        raise ValueError("grid angular_count %d does not match signal length %d"
                         % (grid.angular_count, g.shape[-1]))
    if engine not in ENGINES:
        raise ValueError("engine must be 'fft' or 'direct', got %r" % (engine,))  # core.py:357-358
    if max_terms < 1:
        raise ValueError("max_terms must be >= 1")
    if threshold is not None and not 0.0 < threshold <= 1.0:
        raise ValueError("threshold must lie in (0, 1]")
    if engine == "direct" and g.shape[-1] > 8192:
        raise NotImplementedError("engine 'direct' (O(M N^2) literal sums) supports N <= 8192")


def _build(grid, n, engine, rec, count, initial, remainder):
    """Decomposition from device step records.  The frozen dataclasses are
    filled without re-running __post_init__: the device produced the values
    from a validated grid."""
    rec = rec[:count]
    radius = rec["radius"].tolist()
    j = rec["j"].tolist()
    a = (rec["a_re"] + 1j * rec["a_im"]).tolist()
    c = (rec["c_re"] + 1j * rec["c_im"]).tolist()
    res = rec["residual"].tolist()
    new, sa = object.__new__, object.__setattr__
    P, S = ParameterPoint, DecompositionStep
    steps = []
    for k in range(count):
        pt = new(P)
        sa(pt, "__dict__", {"radius": radius[k], "angle_index": j[k], "value": a[k]})
        st = new(S)
        sa(st, "__dict__", {"point": pt, "coefficient": c[k], "residual_energy": res[k]})
        steps.append(st)
    return Decomposition(tuple(steps), grid, n, float(initial), engine, remainder=remainder,
                         step_flags=tuple(rec["flags"].tolist()),
                         margins=tuple(rec["margin"].astype(np.float64).tolist()))


def decompose(g, grid, max_terms=10, threshold=None, engine="fft", dc_first=False,
              parallel=False):
    """Greedy AFD of G over the grid on the B200 (core.py:317-391).

    Same contract as the reference: stops after ``max_terms`` steps, once
    residual <= threshold * initial energy, or at an exactly zero residual;
    empty decomposition for a zero-energy input.  The whole loop (forward
    transform, fused field + argmax, remainder update, energy, stop rules)
    runs device-resident as one CUDA graph.
    """
    g = _as_signal(g)
    _check_decompose_args(g, grid, max_terms, threshold, engine)
    return decompose_batch(g[None, :], grid, max_terms, threshold, engine, dc_first,
                           parallel, _validated=True)[0]


def decompose_batch(signals, grid, max_terms=10, threshold=None, engine="fft", dc_first=False,
                    parallel=False, _validated=False):
    """``decompose`` for a batch of independent signals ([B, N]) in one pass.

    Entry b equals ``decompose(signals[b], ...)`` exactly.
    """
    sig = np.asarray(signals, dtype=np.complex128)
    if sig.ndim != 2:
        raise ValueError("signals must be 2-d [batch, N], got shape %r" % (sig.shape,))
    if not _validated:
        # _as_signal on every row, vectorised (same checks, same messages)
        if sig.shape[0] and not _is_pow2(sig.shape[1], 8):
            raise ValueError("signal length must be a power of two >= 8, got %d" % sig.shape[1])
        if not np.all(np.isfinite(sig)):
            raise ValueError("signal contains non-finite samples")
        _check_decompose_args(sig, grid, max_terms, threshold, engine)
    b, n = sig.shape
    plan = _engine().get_plan(grid.radii, n, batch=b, engine=1 if engine == "direct" else 0,
                              fast=_FAST_LEVEL.get(engine, 0))
    rec, counts, initial, rem, _, _ = plan.decompose_host(sig, int(max_terms), threshold,
                                                          dc_first)
    if b == 1:
        return [_build(grid, n, engine, rec[0], int(counts[0]), initial[0], rem[0])]
    # tens of thousands of small objects: the cyclic GC's generation scans
    # would double the build time (c3: 1024 x 20 steps), and none of them
    # can be part of a cycle
    gc_was = gc.isenabled()
    gc.disable()
    try:
        return _build_batch(grid, n, engine, rec, counts, initial, rem)
    finally:
        if gc_was:
            gc.enable()


def _build_batch(grid, n, engine, rec, counts, initial, rem):
    """_build for every signal of a batch, the record fields converted to
    Python scalars once for the whole batch."""
    radius = rec["radius"].tolist()
    j = rec["j"].tolist()
    a = (rec["a_re"] + 1j * rec["a_im"]).tolist()
    c = (rec["c_re"] + 1j * rec["c_im"]).tolist()
    res = rec["residual"].tolist()
    flags = rec["flags"].tolist()
    margins = rec["margin"].astype(np.float64).tolist()
    counts = counts.tolist()
    initial = initial.tolist()
    new, sa = object.__new__, object.__setattr__
    P, S = ParameterPoint, DecompositionStep
    out = []
    for i, count in enumerate(counts):
        ri, ji, ai, ci, si = radius[i], j[i], a[i], c[i], res[i]
        steps = []
        for k in range(count):
            pt = new(P)
            sa(pt, "__dict__", {"radius": ri[k], "angle_index": ji[k], "value": ai[k]})
            st = new(S)
            sa(st, "__dict__", {"point": pt, "coefficient": ci[k], "residual_energy": si[k]})
            steps.append(st)
        out.append(Decomposition(tuple(steps), grid, n, initial[i], engine, remainder=rem[i],
                                 step_flags=tuple(flags[i][:count]),
                                 margins=tuple(margins[i][:count])))
    return out


# ---------------------------------------------------------------------------
# basis, reconstruction, errors (core.py:394-460)
# ---------------------------------------------------------------------------

def tm_basis_samples(poles, n):
    """k-th orthonormal rational basis function for the pole prefix (core.py:394-408)."""
    values = [_pole_value(a) for a in poles]
    if not values:
        raise ValueError("need at least one pole")
    p = _plan(int(n))
    b = p.atom(0, values[-1], norm=_kernel_norm(values[-1]))
    for a in values[:-1]:
        b = p.atom(3, a, g=b)
    return _host(b)


def _steps_device(d, n_terms, plan):
    rec = np.zeros((1, max(n_terms, 1)), dtype=_capi.STEP_DTYPE)
    for k, s in enumerate(d.steps[:n_terms]):
        rec[0, k] = (0, s.point.angle_index, s.point.radius, s.point.value.real,
                     s.point.value.imag, s.coefficient.real, s.coefficient.imag,
                     s.residual_energy, 0, 0)
    t = _torch()
    steps = t.from_numpy(rec.view(np.uint8).reshape(1, rec.shape[1], -1)).to(plan.device)
    count = t.tensor([n_terms], dtype=t.int32, device=plan.device)
    return steps, count


def _trace(d, g, n_terms):
    eng = _engine()
    plan = _plan(d.n_samples)
    steps, count = _steps_device(d, n_terms, plan)
    dec = eng.DeviceDecomposition(steps=steps, n_steps=count, initial=None, remainder=None)
    norms = _torch().tensor([[_kernel_norm(s.point.value) for s in d.steps[:n_terms]] or [0.0]],
                            dtype=_torch().float64)
    errors, recon = plan.error_trace(_to_dev(g, plan), dec, norms=norms)
    return _host(errors)[0][:n_terms], _host(recon)[0]


def reconstruct(decomposition, n_terms):
    """Partial sum S_n over the first n recorded atoms (core.py:411-427)."""
    steps = decomposition.steps
    n_terms = int(n_terms)
    if not 0 <= n_terms <= len(steps):
        raise ValueError("term count %d outside 0..%d" % (n_terms, len(steps)))
    n = decomposition.n_samples
    if n_terms == 0:
        return np.zeros(n, dtype=np.complex128)
    return _trace(decomposition, np.zeros(n, dtype=np.complex128), n_terms)[1]


def relative_error(g, s):
    """||G - S||^2 / ||G||^2 (core.py:430-439)."""
    g = _as_signal(g)
    s = _as_signal(s)
    if g.shape != s.shape:
        raise ValueError("length mismatch: %d vs %d" % (g.shape[0], s.shape[0]))
    p = _plan(g.shape[0])
    gd, sd = _to_dev(g, p), _to_dev(s, p)
    eg = float(_host(p.energy(gd))[0])
    es = float(_host(p.energy_diff(gd, sd))[0])
    if eg == 0.0:
        raise ValueError("relative error undefined for a zero-energy reference")
    return float(es / eg)


def error_trace(decomposition, g):
    """Relative errors of the partial sums, entry i for the (i+1)-term sum (core.py:442-460)."""
    g = _as_signal(g)
    if g.shape[0] != decomposition.n_samples:
        raise ValueError("signal length %d does not match decomposition %d"
                         % (g.shape[0], decomposition.n_samples))
    if not decomposition.steps:
        return []
    errs, _ = _trace(decomposition, g, len(decomposition.steps))
    return [float(e) for e in errs]
