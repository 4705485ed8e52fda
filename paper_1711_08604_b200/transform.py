"""Reference-compatible transforms (``fastafd.transform``), computed on the B200.

Same names, contracts and errors as ``/root/reference/pkg/src/fastafd/
transform.py``; the numbers come from the exact-DIT kernels of
``libafd_b200.so`` (bit-identical to the reference's radix-2 butterflies).
"""

from __future__ import annotations

import numpy as np

__all__ = ["bit_reverse_permute", "dft_forward", "dft_inverse", "weighted_inverse",
           "weighted_inverse_grid"]


def _checked_length(x):
    """1-d power-of-two buffer check (transform.py:38-45)."""
    x = np.asarray(x)
    if x.ndim != 1:
        raise ValueError("expected a 1-d buffer, got shape %r" % (x.shape,))
    n = x.shape[0]
    if n < 2 or n & (n - 1):
        raise ValueError("length must be a power of two >= 2, got %d" % n)
    return x, n


def _checked_radius(r):
    r = float(r)
    if not 0.0 <= r < 1.0:
        raise ValueError("radius must satisfy 0 <= r < 1, got %g" % r)
    return r


def _bitrev(n):
    bits = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def bit_reverse_permute(x):
    """output[j] = x[bitrev(j)] (transform.py:96-103); index plumbing, no arithmetic."""
    x, n = _checked_length(x)
    return x[_bitrev(n)]


def _plan(n, radii=(0.0,)):
    from . import engine
    if n < 8:
        raise NotImplementedError("the device transforms need N >= 8, got %d" % n)
    return engine.get_plan(radii, n)


def _run(kind, x):
    import torch
    x, n = _checked_length(x)
    p = _plan(n)
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(p.device)
    out = p.dft_forward(t) if kind == "fwd" else p.dft_inverse(t)
    return out[0].cpu().numpy()


def dft_forward(x):
    """Unnormalised forward DFT (transform.py:106-124)."""
    return _run("fwd", x)


def dft_inverse(c):
    """1/N inverse DFT (transform.py:127-134)."""
    return _run("inv", c)


def weighted_inverse(c, r):
    """Single-radius weighted inverse (transform.py:166-182)."""
    return weighted_inverse_grid(c, (r,))[0]


def weighted_inverse_grid(c, radii):
    """(M, N) weighted inverse rows, identical per row to single calls (transform.py:185-201)."""
    import torch
    c, n = _checked_length(c)
    radii = tuple(_checked_radius(r) for r in radii)
    if not radii:
        raise ValueError("need at least one radius")
    p = _plan(n, radii)
    t = torch.from_numpy(np.ascontiguousarray(c, dtype=np.complex128)).to(p.device)
    return p.field(t).cpu().numpy()
