"""The reference's "direct" engine (``fastafd.oracle``), on the device.

``field_direct(g, grid)`` mirrors ``oracle.field_direct`` (oracle.py:51-73):
all grid inner products <G, e_a> by literal O(N) summation per point, as
the circular correlation of G with the sampled normalised kernel rows.
``core.decompose(..., engine="direct")`` runs the whole decomposition with
it.  Agreement with the reference is to its own engine tolerance (1e-9,
identical poles); see csrc/afd_direct.cuh.
"""

from __future__ import annotations

import numpy as np

__all__ = ["field_direct"]


def field_direct(g, grid):
    """(M, N) field by direct summation (oracle.py:51-73), computed on the B200."""
    import torch

    from . import core, engine
    g = core._as_signal(g)
    if grid.angular_count != g.shape[0]:
        raise ValueError("grid angular_count %d does not match signal length %d"
                         % (grid.angular_count, g.shape[0]))
    plan = engine.get_plan(grid.radii, g.shape[0], engine=1)
    return plan.field_direct(torch.from_numpy(g).to(plan.device)).cpu().numpy()
