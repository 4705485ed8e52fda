"""Seeded synthetic inputs for the BASELINE configurations (host side).

BASELINE.json names five workloads c0..c4; no public dataset is involved, the
generators below restate them.  All randomness comes from
``np.random.Generator(np.random.Philox(seed))``, the PRNG family the
reference uses for its own random signals (``signals.py:86``).

* c0..c1, c3, c4: pole sums ``G(z) = sum_j c_j / (1 - conj(b_j) z)`` sampled on
  ``z_m = exp(2 pi i m / N)``; ``b_j = R sqrt(U) e^{2 pi i V}`` is area-uniform
  in ``|b| < R``, ``c_j`` is a standard complex Gaussian.  Draw order: P
  uniforms U, P uniforms V, P real normals, P imaginary normals.
* c2: real cosine series ``sum_{k=1..64} (1/k) cos(k t + phi_k) + 0.01 n``
  (phi_k = 2 pi U_k drawn first, then the N noise normals), projected to the
  Hardy space by the analytic projection (``core.py:201-231``), on the GPU.

The radius grid for every config is ``r_m = m / M``, m = 0..M-1.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "CONFIGS", "pole_sum", "cosine_series", "radii_for",
           "signal_for"]


@dataclass(frozen=True)
class Workload:
    name: str
    n: int              # samples = angular grid size N
    m: int              # radii M
    steps: int          # AFD steps
    poles: int          # P (pole-sum inputs), 0 for the cosine series
    radius: float       # R, pole radius bound
    seed: int
    batch: int = 1      # independent signals (c3)
    real: bool = False  # real input needing the analytic projection (c2)

    @property
    def evals_per_decomposition(self):
        return self.batch * self.m * self.n * self.steps


CONFIGS = {
    "c0": Workload("c0", 1024, 100, 10, 8, 0.9, 0),
    "c1": Workload("c1", 4096, 512, 30, 32, 0.95, 1),
    "c2": Workload("c2", 65536, 4096, 50, 0, 0.0, 2, real=True),
    "c3": Workload("c3", 4096, 1024, 20, 16, 0.9, 1000, batch=1024),
    "c4": Workload("c4", 1 << 20, 16384, 20, 128, 0.99, 4),
}


def _rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def pole_sum(n, poles, radius, seed):
    """G(z_m) = sum_j c_j / (1 - conj(b_j) z_m), complex128, length n."""
    rng = _rng(seed)
    u = rng.uniform(size=poles)
    v = rng.uniform(size=poles)
    cre = rng.standard_normal(poles)
    cim = rng.standard_normal(poles)
    b = radius * np.sqrt(u) * np.exp(2j * np.pi * v)
    c = cre + 1j * cim
    z = np.exp(2j * np.pi * np.arange(n) / n)
    g = np.zeros(n, dtype=np.complex128)
    for j in range(poles):
        g = g + c[j] / (1.0 - np.conj(b[j]) * z)
    return g


def cosine_series(n, seed, terms=64, noise=0.01):
    """Real x(t_m) = sum_k (1/k) cos(k t_m + phi_k) + noise * N(0,1)."""
    rng = _rng(seed)
    phi = 2.0 * np.pi * rng.uniform(size=terms)
    nz = rng.standard_normal(n)
    t = 2.0 * np.pi * np.arange(n) / n
    x = np.zeros(n, dtype=np.float64)
    for k in range(1, terms + 1):
        x = x + (1.0 / k) * np.cos(k * t + phi[k - 1])
    return x + noise * nz


def radii_for(m):
    """r_m = m / M, m = 0..M-1 (includes the all-equal r = 0 row)."""
    return tuple(k / m for k in range(m))


def signal_for(cfg, index=0):
    """Input of signal `index` of workload `cfg` (real samples for c2)."""
    w = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    if w.real:
        return cosine_series(w.n, w.seed + index)
    return pole_sum(w.n, w.poles, w.radius, w.seed + index)
