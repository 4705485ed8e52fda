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

__all__ = ["shard_bounds", "radius_shard_bounds", "live_powers", "expected_twopass",
           "expected_tier", "FAST_TIER_COST", "decompose_sharded",
           "decompose_batch_sharded", "ShardedRunner"]


def shard_bounds(count, rank, world):
    """Contiguous, balanced [lo, hi) block of `count` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank %d outside world of %d" % (rank, world))
    return (count * rank) // world, (count * (rank + 1)) // world


def live_powers(radii, n):
    """Per radius, the number of leading entries of its r^l row (the
    reference's sequential np.cumprod fold, transform.py:147-150) that are
    not exactly +0 — the entries the exact large-N field loads (pw_len on the
    device).  Only r <= 0.5 ever reaches zero: for r > 0.5 the fold sticks at
    a subnormal (k 2^-1074 r rounds back to k 2^-1074), so those rows are
    live to the end."""
    r = np.asarray(radii, dtype=np.float64)
    live = np.full(r.shape, int(n), dtype=np.int64)
    idx = np.nonzero(r <= 0.5)[0]
    v = np.ones(idx.size)
    rr = r[idx]
    for l in range(1, int(n)):
        if idx.size == 0:
            break
        v = v * rr
        z = v == 0.0
        if z.any():
            live[idx[z]] = l
            keep = ~z
            idx, v, rr = idx[keep], v[keep], rr[keep]
    return live


def expected_twopass(radii, n, onchip=4096):
    """Rows the pruned fast field (csrc/afd_pruned.cuh) is expected to leave
    to the two-pass path: those whose weight tail r^l, l >= `onchip`,
    exceeds 2^-64 of the largest kept term even for a flat spectrum,
    r^L / (1 - r) > 2^-64.  (The device decides per step from the actual
    spectrum; this is the plan-time estimate used to balance shards.)"""
    r = np.asarray(radii, dtype=np.float64)
    with np.errstate(divide="ignore"):
        lt = onchip * np.log2(np.where(r > 0.0, r, 1.0)) - np.log2(1.0 - r)
    return (r > 0.0) & (lt > -64.0)


# Spectrum terms per tier of the pruned fast field (csrc/afd_pruned.cuh: 32,
# 64, 128 in registers, 256 ... 4096 as on-chip transforms) and the measured
# cost of one row relative to a 1024-point row (c4, N = 2^20, one B200:
# 1.03, 1.18, 1.53, 1.98, 2.25, 2.55, 3.47 us per row; two-pass 7.5 us;
# profiles/r02/tier_kernels_c4_v13.txt).
FAST_TIERS = (32, 64, 128, 256, 512, 1024, 4096)
FAST_TIER_COST = {32: 0.40, 64: 0.46, 128: 0.60, 256: 0.78, 512: 0.88, 1024: 1.0, 4096: 1.36,
                  None: 2.9}


def expected_tier(radii, n):
    """Per radius, the spectrum terms L of the tier the pruned fast field is
    expected to evaluate the row from — the first L in FAST_TIERS with
    r^L / (1 - r) <= 2^-64 (a flat spectrum) — or `n` for the two-pass rows
    (estimate_tier_rows in csrc/afd_capi.cu; the device decides per step
    from the actual spectrum)."""
    r = np.asarray(radii, dtype=np.float64)
    out = np.full(r.shape, int(n), dtype=np.int64)
    with np.errstate(divide="ignore"):
        lr, l1r = np.log2(np.where(r > 0.0, r, 1.0)), np.log2(1.0 - r)
    for L in reversed(FAST_TIERS):
        out[(r == 0.0) | (L * lr - l1r <= -64.0)] = L
    return out


def radius_shard_bounds(radii, n, rank, world, exact=True):
    """Contiguous radius block [m0, m1) of `rank` balanced by field cost.

    Large N (> 8192):
    * exact field: a row costs its 32 B per eval of row-batch intermediate
      plus 8 B per live r^l entry (live_powers) — rows with r <= 0.5 are
      cheaper;
    * fast field: a row is evaluated from as many spectrum terms as its
      weight tail needs (the pruned field's tiers) and costs accordingly —
      the register tiers (r <= 0.7) under half a 1024-point row, the few
      radii closest to 1 (two-pass) three times as much: rows weigh
      FAST_TIER_COST[expected_tier].
    Blocks are cut at equal cumulative cost, so the high-radius rank does
    not set the step time.  On-chip N: every row costs the same and this is
    shard_bounds.  Blocks stay rank-ordered and non-empty, so the
    lowest-flat-index tie rule holds."""
    m = len(radii)
    if n <= 8192 or world == 1:
        return shard_bounds(m, rank, world)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank %d outside world of %d" % (rank, world))
    if exact:
        cost = 32.0 + 8.0 * live_powers(radii, n) / float(n)
    else:
        tier = expected_tier(radii, n)
        cost = np.full(m, FAST_TIER_COST[None])
        for L in FAST_TIERS:
            cost[tier == L] = FAST_TIER_COST[L]
    cum = np.concatenate([[0.0], np.cumsum(cost)])

    def cut(p):
        if p <= 0:
            return 0
        if p >= world:
            return m
        b = int(np.searchsorted(cum, cum[-1] * p / world))
        if b > 0 and abs(cum[b - 1] - cum[-1] * p / world) <= abs(cum[b] - cum[-1] * p / world):
            b -= 1
        return min(max(b, p), m - (world - p))
    return cut(rank), cut(rank + 1)


def _all_gather(out, t, group):
    """One all-gather of every rank's candidates, chosen by backend (every
    rank issues the same collective): all_gather_into_tensor on NCCL, the
    list form elsewhere (gloo)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t, group=group)


def _default_plan(radii, n, batch, m0, m1, device, engine_name="fft"):
    from . import engine
    return engine.get_plan(radii, n, batch=batch, m0=m0, m1=m1, device=device,
                           engine=1 if engine_name == "direct" else 0,
                           fast={"fft-fast": 1, "fft-fast-margins": 2}.get(engine_name, 0))


_COMMS = {}


def library_comm(group, device):
    """The library's own NCCL communicator over `group` (cached per group):
    rank 0 draws the NCCL unique id, torch.distributed broadcasts it."""
    import torch.distributed as dist
    from . import engine
    key = (id(group), str(device))
    c = _COMMS.get(key)
    if c is None:
        obj = [engine.Comm.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        c = engine.Comm(obj[0], dist.get_world_size(group), dist.get_rank(group),
                        device.index)
        _COMMS[key] = c
    return c


class ShardedRunner:
    """The radius-sharded decomposition loop of one rank.

    Per AFD step: the rank's field + argmax over its rows (select_local), an
    all-gather of the 32-byte candidates of all ranks (rank-major, so the
    lowest flat index still wins ties), then the identical replicated
    update + energy + next spectrum (apply_step).  The host issues the steps
    without ever synchronising; once a signal's stop rule fires its kernels
    are no-ops.  Reusable: ``run`` may be called repeatedly (benchmarks).

    On an NCCL group with CUDA plans the whole loop is device-resident: the
    library captures it, all-gathers included, into one CUDA graph
    (afd_decompose_sharded over the library's own communicator).  Otherwise
    (gloo, CPU stand-in plans) the host issues it step by step."""

    def __init__(self, plan, batch, max_terms, threshold=None, dc_first=False, group=None):
        import torch
        import torch.distributed as dist
        self.plan, self.batch, self.max_terms = plan, int(batch), int(max_terms)
        self.threshold, self.dc_first, self.group = threshold, bool(dc_first), group
        self.world = dist.get_world_size(group)
        dev = plan.device
        self.steps = torch.zeros((self.batch, self.max_terms, _capi.STEP_DTYPE.itemsize),
                                 dtype=torch.uint8, device=dev)
        self.gathered = torch.empty((self.world, self.batch, 32), dtype=torch.uint8,
                                    device=dev)
        self.cpu = dist.get_backend(group) != "nccl" and dev.type == "cuda"
        self.fin = None
        self.device_loop = (dist.get_backend(group) == "nccl" and dev.type == "cuda" and
                            hasattr(plan, "decompose_sharded"))
        if self.device_loop:
            self.comm = library_comm(group, dev)
            self.out = plan.alloc_outputs(self.batch, self.max_terms)

    def run(self, g):
        """Decompose g ([batch, N], on the plan's device) over all ranks."""
        p = self.plan
        if self.device_loop:
            o = p.decompose_sharded(self.comm, g, self.max_terms, self.threshold,
                                    self.dc_first, out=self.out)
            self.steps = o.steps
            self.fin = (o.n_steps, o.initial, o.remainder, None)
            return self.fin
        p.sharded_begin(g)
        for k in range(self.max_terms):
            local = p.select_local(k, self.dc_first, self.batch)           # [B, 32]
            if self.cpu:  # gloo: exchange through host memory
                host = self.gathered.cpu()
                _all_gather(host, local.cpu().contiguous(), self.group)
                self.gathered.copy_(host)
            else:
                _all_gather(self.gathered, local.contiguous(), self.group)
            cands = self.gathered.permute(1, 0, 2).contiguous()           # [B, P, 32]
            p.apply_step(k, self.max_terms, self.threshold, self.dc_first, cands, self.steps)
        self.fin = p.sharded_finish(self.batch)
        return self.fin

    def host_records(self):
        """(step records [batch, max_terms], n_steps [batch]) of the last run."""
        rec = self.steps.cpu().numpy().view(_capi.STEP_DTYPE)[..., 0]
        return rec, self.fin[0].cpu().numpy()


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
    m0, m1 = radius_shard_bounds(grid.radii, n, rank, world,
                                 exact=not engine_name.startswith("fft-fast"))
    if plan_factory is None:
        plan = _default_plan(grid.radii, n, b, m0, m1, device, engine_name)
    else:
        plan = plan_factory(grid.radii, n, b, m0, m1, device)
    dev = plan.device
    g = torch.from_numpy(sig).to(dev)
    runner = ShardedRunner(plan, b, max_terms, threshold, dc_first, group)
    n_steps, initial, rem, _ = runner.run(g)
    rec = runner.steps.cpu().numpy().view(_capi.STEP_DTYPE)[..., 0]
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
