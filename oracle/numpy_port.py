"""The reference's selection step as numpy — TEST / BASELINE INFRASTRUCTURE ONLY.

A numpy restatement of the reference's hot step (one AFD step's grid field
and argmax): the cumprod radius tables and bit-reversed gather of
``transform._radius_tables`` / ``weighted_inverse_grid``
(reference pkg/src/fastafd/transform.py:137-201), the stage loop of
``transform._butterflies`` (transform.py:73-93) over the whole M x N array,
the scale, and ``core.maximal_selection``'s |F|^2 + first argmax
(core.py:285-300).  It runs the same numpy operations, so it computes the
same bits as the reference (and as ``afd_oracle.c``), at the reference's
own speed: ``bench.py`` times it single-threaded on the GPU box as the
reference numpy baseline (the reference package itself is not on that box).
Only ``tests/`` and ``bench.py`` import this module.
"""

from __future__ import annotations

import numpy as np


def _bitrev(n):
    k = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.int64)
    for b in range(k):
        out |= ((idx >> b) & 1) << (k - 1 - b)
    return out


class Tables:
    """Per-(radii, N) tables, built once like the reference's plan cache."""

    def __init__(self, radii, n):
        self.n = int(n)
        self.rev = _bitrev(self.n)
        self.w_inv = np.conj(np.exp(-2j * np.pi * np.arange(self.n // 2) / self.n))
        r = np.asarray(radii, dtype=np.float64)
        rows = np.empty((r.shape[0], self.n))
        rows[:, 0] = 1.0
        rows[:, 1:] = r[:, None]
        np.cumprod(rows, axis=1, out=rows)
        self.powers = np.ascontiguousarray(rows[:, self.rev])
        self.scales = np.sqrt(1.0 - r * r) / (self.n * (1.0 - r ** self.n))


def field(t, c):
    """The M x N weighted inverse grid for spectrum c (numpy, in place)."""
    y = np.ascontiguousarray(t.powers * c[t.rev], dtype=np.complex128)
    n = t.n
    span = 2
    while span <= n:
        h = span // 2
        blk = y.reshape(-1, span)
        prod = blk[:, h:] * t.w_inv[:: n // span]
        blk[:, h:] = blk[:, :h] - prod
        blk[:, :h] += prod
        span *= 2
    y *= t.scales[:, None]
    return y


def select(t, c):
    """(s, j, |F|^2, F) of the first maximum of the grid for spectrum c."""
    y = field(t, c)
    mag = y.real * y.real + y.imag * y.imag
    flat = int(np.argmax(mag))
    s, j = divmod(flat, t.n)
    return s, j, float(mag.flat[flat]), complex(y.flat[flat])
