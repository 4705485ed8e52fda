"""Multi-GPU AFD: radius sharding with one tiny collective per step.

SURVEY.md §8(e).  Within a step the M x N field is M independent rows, so
rank p owns the contiguous radius block ``shard_bounds(M, p, P)``; flat
indices s*N + j are then rank-ordered, which preserves the reference's
"lowest flat index wins" tie rule (core.py:299).  Every rank keeps a full
replica of the remainder G_k and runs the (cheap, deterministic) update and
forward transform itself, so the remainders stay bit-identical across ranks
and no broadcast of G or a_k is needed: the only exchange per step is an
all-gather of one 32-byte candidate (|F|^2, flat, F) per rank and signal —
NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests — after which each
rank reduces the P candidates on device with the same first-maximum rule.

The loop always issues ``max_terms`` steps without reading anything back:
once a signal's stop rule fires (core.py:386-389) its kernels turn into
no-ops, so the host never synchronises inside the loop.

Independent signals (BASELINE c3) need no collective at all: shard the
batch with ``shard_bounds(B, p, P)`` and call ``core.decompose_batch``.
"""

from __future__ import annotations

import numpy as np

from . import _capi

__all__ = ["shard_bounds", "decompose_sharded", "decompose_batch_sharded"]


def shard_bounds(count, rank, world):
    """Contiguous, balanced [lo, hi) block of `count` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank %d outside world of %d" % (rank, world))
    return (count * rank) // world, (count * (rank + 1)) // world


def _all_gather(out, t, group):
    """all_gather_into_tensor where the backend has it (NCCL), else the list form (gloo)."""
    import torch.distributed as dist
    try:
        dist.all_gather_into_tensor(out, t, group=group)
    except (RuntimeError, NotImplementedError, ValueError):
        dist.all_gather(list(out.unbind(0)), t, group=group)


def _default_plan(radii, n, batch, m0, m1, device):
    from . import engine
    return engine.get_plan(radii, n, batch=batch, m0=m0, m1=m1, device=device)


def decompose_sharded(signals, grid, max_terms=10, threshold=None, dc_first=False, group=None,
                      device=None, plan_factory=None, engine_name="fft"):
    """Radius-sharded ``decompose_batch`` over the ranks of ``group``.

    Every rank passes the same signals ([B, N] or [N]) and grid and gets the
    same list of Decompositions, identical to the single-GPU result.
    ``plan_factory(radii, n, batch, m0, m1, device)`` returns the per-rank
    plan (default: the CUDA plan); tests inject an oracle-backed stand-in.
    """
    import torch
    import torch.distributed as dist

    from . import core

    sig = np.asarray(signals, dtype=np.complex128)
    if sig.ndim == 1:
        sig = sig[None, :]
    for row in sig:
        core._as_signal(row)
    core._check_decompose_args(sig, grid, max_terms, threshold, engine_name)
    b, n = sig.shape
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    m = len(grid.radii)
    if world > m:
        raise ValueError("more ranks (%d) than radii (%d)" % (world, m))
    m0, m1 = shard_bounds(m, rank, world)
    plan = (plan_factory or _default_plan)(grid.radii, n, b, m0, m1, device)
    dev = plan.device
    g = torch.from_numpy(sig).to(dev)
    plan.sharded_begin(g)
    steps = torch.zeros((b, max_terms, _capi.STEP_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    gathered = torch.empty((world, b, 32), dtype=torch.uint8, device=dev)
    for k in range(max_terms):
        local = plan.select_local(k, dc_first, b)                    # [B, 32]
        _all_gather(gathered, local.contiguous(), group)
        cands = gathered.permute(1, 0, 2).contiguous()               # [B, P, 32] rank-major
        plan.apply_step(k, max_terms, threshold, dc_first, cands, steps)
    n_steps, initial, rem, _ = plan.sharded_finish(b)
    rec = steps.cpu().numpy().view(_capi.STEP_DTYPE)[..., 0]
    counts = n_steps.cpu().numpy()
    init = initial.cpu().numpy()
    remh = rem.cpu().numpy()
    return [core._build(grid, n, engine_name, rec[i], int(counts[i]), init[i], remh[i].copy())
            for i in range(b)]


def decompose_batch_sharded(signals, grid, max_terms=10, threshold=None, dc_first=False,
                            group=None, engine_name="fft", gather=True, decompose_fn=None):
    """Signal-sharded ``core.decompose_batch`` (BASELINE c3).

    Rank p decomposes the contiguous block ``shard_bounds(B, p, P)`` of the
    batch on its own GPU — no collective inside the loop.  With ``gather``
    the per-signal Decompositions are all-gathered once at the end, so every
    rank returns the whole batch in order (identical to the single-GPU
    result); otherwise each rank returns its own block.
    ``decompose_fn(signals, grid, max_terms, threshold, dc_first)`` replaces
    the CUDA decomposition (tests inject a CPU stand-in).
    """
    import torch.distributed as dist

    from . import core

    sig = np.asarray(signals, dtype=np.complex128)
    if sig.ndim != 2:
        raise ValueError("signals must be 2-d [batch, N], got shape %r" % (sig.shape,))
    core._check_decompose_args(sig, grid, max_terms, threshold, engine_name)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = shard_bounds(sig.shape[0], rank, world)
    if decompose_fn is None:
        def decompose_fn(x, gr, mt, thr, dc):
            return core.decompose_batch(x, gr, mt, thr, engine_name, dc) if len(x) else []
    local = decompose_fn(sig[lo:hi], grid, max_terms, threshold, dc_first)
    if not gather:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return [d for part in parts for d in part]
