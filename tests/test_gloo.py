"""world_size-2 gloo tests of the multi-GPU host logic (CPU):
shard coverage, deterministic rank-ordered OLS-statistics reduction, and the
gather of fixed-size per-scenario report rows with uneven shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_18725_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(rank)
        stats = torch.tensor(rng.normal(size=56), dtype=torch.float64)
        red = D.allreduce_ols_stats(stats)
        n_total = 7
        lo, hi = D.shard_range(n_total, rank, world)
        local = torch.tensor([[float(i)] * 3 for i in range(lo, hi)], dtype=torch.float64)
        full = D.gather_rows(local, n_total)
        q.put((rank, red.numpy(), full.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduce_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    expect = np.random.default_rng(0).normal(size=56) + np.random.default_rng(1).normal(size=56)
    for _, red, full in res:
        np.testing.assert_array_equal(red, expect)  # rank-ordered sum, identical on every rank
        np.testing.assert_array_equal(full[:, 0], np.arange(7.0))
    np.testing.assert_array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("n,world", [(0, 2), (7, 2), (10, 4), (3, 8), (10000, 8)])
def test_shard_range_partitions(n, world):
    got = [D.shard_range(n, r, world) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
    sizes = [h - l for l, h in got]
    assert max(sizes) - min(sizes) <= 1


def test_weighted_shards_cover_and_balance():
    w = np.random.default_rng(0).uniform(100, 2000, size=1000)
    sh = D.weighted_shards(w, 8)
    assert sh[0][0] == 0 and sh[-1][1] == 1000
    loads = [w[l:h].sum() for l, h in sh]
    assert max(loads) / min(loads) < 1.05


def test_lpt_shards_cover_balance_and_order():
    """C5 strong-scaling split: every scenario exactly once, loads within a
    few percent, each rank's list in descending weight (its replay order)."""
    from paper_2512_18725_b200.profiles import gen_synthetic_profiles
    from paper_2512_18725_b200.sweep import c5_scenarios, expected_requests

    w = [expected_requests(s) for s in c5_scenarios(gen_synthetic_profiles(), 2000)]
    for world in (1, 2, 4, 8):
        sh = D.lpt_shards(w, world)
        assert sorted(i for s in sh for i in s) == list(range(len(w)))
        loads = [sum(w[i] for i in s) for s in sh]
        assert max(loads) / min(loads) < 1.01
        for s in sh:
            assert all(w[a] >= w[b] for a, b in zip(s, s[1:]))
    assert D.lpt_shards(w, 8) == D.lpt_shards(list(w), 8)  # deterministic: every rank computes the same split


def _sweep_rows_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        counts = [5, 3]
        local = torch.full((counts[rank], D.SWEEP_ROW), float(rank), dtype=torch.float64)
        blocks = D.gather_sweep_rows(local, counts, backend="gloo")
        q.put((rank, [b.numpy() for b in blocks]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_sweep_rows_uneven():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, blocks in res:
        assert [b.shape[0] for b in blocks] == [5, 3]
        assert (blocks[0] == 0).all() and (blocks[1] == 1).all()
