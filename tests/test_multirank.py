"""Radius-sharded decomposition across 2 ranks (gloo, CPU) == single-process result.

Exercises distributed.decompose_sharded's host logic (shard bounds, the
per-step all-gather of 32-byte candidates, the rank-major merge, the step
loop) with an oracle-backed stand-in for the CUDA plan.
"""

import os
import socket
import warnings

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from conftest import load_golden

warnings.simplefilter("ignore", UserWarning)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_plan import OraclePlan
        from paper_1711_08604_b200 import core, distributed
        g = load_golden("decomp_%s.npz" % case)
        thr = float(g["threshold"])
        grid = core.ParameterGrid(tuple(g["radii"]), g["g"].shape[0])
        ds = distributed.decompose_sharded(
            g["g"], grid, max_terms=int(g["max_terms"]),
            threshold=None if np.isnan(thr) else thr, dc_first=bool(g["dc_first"]),
            plan_factory=OraclePlan)
        d = ds[0]
        out_q.put((rank, [s.point.angle_index for s in d.steps],
                   [s.point.radius for s in d.steps], [s.coefficient for s in d.steps],
                   [s.residual_energy for s in d.steps], d.remainder))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("c0", 2), ("f2_dc", 2), ("f1_thr", 3)])
def test_radius_sharded_equals_reference(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_golden("decomp_%s.npz" % case)
    for rank, j, radius, coeff, resid, rem in res:
        assert j == list(g["j"]), rank
        assert radius == list(g["radius"]), rank
        assert coeff == list(g["coeff"]), rank
        assert resid == list(g["residual"]), rank
        assert np.array_equal(rem, g["remainder"]), rank


def test_shard_bounds():
    from paper_1711_08604_b200.distributed import shard_bounds
    for m in (1, 7, 100, 16384):
        for world in (1, 2, 3, 8):
            if world > m:
                continue
            blocks = [shard_bounds(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert max(h - l for l, h in blocks) - min(h - l for l, h in blocks) <= 1


def test_live_powers_match_the_cumprod_fold():
    """live_powers = count of leading nonzero entries of the reference's
    np.cumprod rows (transform.py:145-149)."""
    from paper_1711_08604_b200.distributed import live_powers
    n = 4096
    radii = np.array([0.0, 0.01, 0.1, 0.25, 0.3, 0.4999, 0.5, 0.5001, 0.9, 0.99])
    powers = np.empty((len(radii), n))
    powers[:, 0] = 1.0
    powers[:, 1:] = radii[:, None]
    np.cumprod(powers, axis=1, out=powers)
    expect = [int(np.argmax(row == 0.0)) if (row == 0.0).any() else n for row in powers]
    assert list(live_powers(radii, n)) == expect
    assert all(np.all(row[e:] == 0.0) for row, e in zip(powers, expect))


def test_radius_shard_bounds_balance_the_exact_field():
    """Exact large-N shards: contiguous, rank-ordered, non-empty, covering,
    and balanced in field cost (32 B + 8 B per live r^l entry per eval) to
    within a row; fast mode balances the pruned field's per-tier row costs;
    on-chip N falls back to row counts."""
    from paper_1711_08604_b200 import workloads as W
    from paper_1711_08604_b200.distributed import (FAST_TIER_COST, expected_tier,
                                                   expected_twopass, live_powers,
                                                   radius_shard_bounds, shard_bounds)
    n, m = 1 << 16, 4096
    radii = W.radii_for(m)
    cost = 32.0 + 8.0 * live_powers(radii, n) / n
    for world in (2, 3, 8):
        blocks = [radius_shard_bounds(radii, n, r, world) for r in range(world)]
        assert blocks[0][0] == 0 and blocks[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
        assert all(h > l for l, h in blocks)
        share = [cost[l:h].sum() for l, h in blocks]
        assert max(share) - min(share) <= 2 * cost.max()
        fast = [radius_shard_bounds(radii, n, r, world, exact=False) for r in range(world)]
        assert fast[0][0] == 0 and fast[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(fast, fast[1:]))
        tier = expected_tier(radii, n)
        assert np.array_equal(tier == n, expected_twopass(radii, n))
        w = np.array([FAST_TIER_COST[None if t == n else int(t)] for t in tier])
        share = [w[l:h].sum() for l, h in fast]
        assert max(share) - min(share) <= 2 * w.max()
        assert [radius_shard_bounds(radii, 4096, r, world) for r in range(world)] == \
            [shard_bounds(m, r, world) for r in range(world)]
    # tiers by radius: r^L / (1 - r) <= 2^-64 at L = 32, 64, 128, 256, 512, 1024, 4096
    assert list(expected_tier((0.0, 0.2, 0.25, 0.3, 0.49, 0.55, 0.69, 0.75, 0.83, 0.9, 0.95, 0.97,
                               0.985, 0.99), n)) == [32, 32, 64, 64, 64, 128, 128, 256, 256, 512,
                                                     1024, 4096, 4096, n]
    tiny = (0.1, 0.2, 0.9)
    assert [radius_shard_bounds(tiny, n, r, 3) for r in range(3)] == [(0, 1), (1, 2), (2, 3)]


def _batch_worker(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_08604_b200 import core, distributed, workloads as W
        n, radii = 128, tuple(i / 16 for i in range(16))
        sig = np.stack([W.pole_sum(n, 4, 0.9, 50 + s) for s in range(7)])
        grid = core.ParameterGrid(radii, n)

        def oracle_batch(x, gr, mt, thr, dc):
            # CPU stand-in for core.decompose_batch: the oracle's records
            out = []
            for row in x:
                o = O.decompose(row, np.array(gr.radii), max_terms=mt)
                out.append((list(o.steps["j"]), list(o.steps["radius"]),
                            list(o.steps["c_re"] + 1j * o.steps["c_im"]), o.remainder))
            return out

        res = distributed.decompose_batch_sharded(sig, grid, max_terms=4,
                                                  decompose_fn=oracle_batch)
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_signal_sharded_batch_gathers_in_order(world):
    """7 signals over 2 / 3 ranks: every rank gets all 7 results, in batch
    order, each equal to the single-process oracle decomposition."""
    from paper_1711_08604_b200 import workloads as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, radii = 128, np.array([i / 16 for i in range(16)])
    want = [O.decompose(W.pole_sum(n, 4, 0.9, 50 + s), radii, max_terms=4) for s in range(7)]
    for rank, got in res:
        assert len(got) == 7, rank
        for (j, r, c, rem), o in zip(got, want):
            assert j == list(o.steps["j"]) and r == list(o.steps["radius"])
            assert c == list(o.steps["c_re"] + 1j * o.steps["c_im"])
            assert np.array_equal(rem, o.remainder)
