"""Multi-rank host logic of the sample-sharded sweep on CPU:
world size 2 over gloo. Each rank reduces its shard to integer histograms
(here with the oracle, standing in for the per-GPU kernel), the product's
reduce_counts all-reduces them, and every rank must hold exactly the
full-window histograms — rank-count invariance, bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_05385_b200.distributed import reduce_counts, shard_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _window(seed=5, n=3001, r=6, c=40):
    rng = np.random.default_rng(seed)
    scores = rng.random((n, r))
    cext = np.hstack([rng.integers(0, 2, size=(n, r)).astype(np.float64), np.ones((n, 1))])
    th = rng.random((c, r))
    return scores, cext, th


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        scores, cext, th = _window()
        lo, hi = shard_range(scores.shape[0], rank, world)
        hist, ok = O.eval_hist(scores[lo:hi], cext[lo:hi], th)
        h, k = reduce_counts(torch.from_numpy(hist), torch.from_numpy(ok))
        out[rank] = (h.numpy().copy(), k.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition_exactly():
    for n in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, g, world) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_single_process_reduce_is_identity():
    h = torch.arange(6, dtype=torch.int64).view(2, 3)
    k = torch.tensor([1, 2], dtype=torch.int64)
    h2, k2 = reduce_counts(h, k)
    assert torch.equal(h, h2) and torch.equal(k, k2)


@pytest.mark.timeout(180)
def test_two_rank_gloo_histograms_equal_full_window():
    from oracle import oracle as O

    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    scores, cext, th = _window()
    hist_full, ok_full = O.eval_hist(scores, cext, th)
    for rank in range(world):
        h, k = out[rank]
        assert np.array_equal(h, hist_full) and np.array_equal(k, ok_full)


def _replica_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_05385_b200.replicas import ReplicaStats, aggregate, replica_batches

        mine = replica_batches(10, rank, world)
        # stand-in for the per-GPU serving loop: fixed per-batch latencies
        lat = [1.0 + rank + 0.1 * i for i in range(len(mine))]
        st = ReplicaStats(rank, 256 * len(mine), sum(lat), lat, exits=200 * len(mine),
                          near_ties=rank)
        out[rank] = (mine, aggregate(st))
    finally:
        dist.destroy_process_group()


def test_replica_dispatch_and_aggregation_world2_gloo():
    """Data-parallel serving (replicas only): request batches are
    split round-robin over replicas with no overlap and no loss, and the job's
    numbers are all samples / the slowest replica and p50 over every replica's
    batch latencies, identical on every rank."""
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_replica_worker, args=(world, port, out), nprocs=world, join=True)
    b0, a0 = out[0]
    b1, a1 = out[1]
    assert sorted(b0 + b1) == list(range(10)) and not set(b0) & set(b1)
    assert a0 == a1
    lat = [1.0 + 0.1 * i for i in range(5)] + [2.0 + 0.1 * i for i in range(5)]
    assert a0["samples"] == 2560 and a0["replicas"] == 2
    assert a0["slowest_replica_ms"] == sum(lat[5:])
    assert a0["samples_per_s"] == 2560 / (sum(lat[5:]) / 1e3)
    assert a0["p50_batch_ms"] == float(np.percentile(lat, 50))
    assert a0["exit_rate"] == 2000 / 2560 and a0["near_tie_rows"] == 1
