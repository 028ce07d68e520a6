"""The sharded sweep's GPU path end to end: two ranks (both on
cuda:0, gloo standing in for NCCL) each run the counts-only sweep on their
sample shard, all-reduce the single histogram+correct-count buffer in place,
and finalise on device (ee_finalize_hist). acc/sav must be bit-identical to
one GPU evaluating the whole window, for the diagonal kernel and the generic
path, with the exchange in line and on a side stream (overlap_comm)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_05385_b200 import synth
        from paper_2312_05385_b200.distributed import ShardedSweep
        from paper_2312_05385_b200.graph import find_feasible_sites

        prof = synth.config4_profile()
        sites = find_feasible_sites(prof)
        arrays = synth.config4_window(60_001)
        diag = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
        rnd = (np.arange(64) / 63.0)[np.random.default_rng(3).integers(0, 64, size=(50, 12))]
        sw = ShardedSweep(arrays, sites, prof, rank=rank, world=world)
        res = [sw.evaluate_many(th) for th in (diag, rnd)]
        # exchange on a side stream (overlap_comm), results read after join()
        comm = torch.cuda.Stream()
        ov = ShardedSweep(arrays, sites, prof, rank=rank, world=world, overlap_comm=True,
                          comm_stream=comm)
        dev = [ov.evaluate_many(th, to_host=False) for th in (diag, rnd, diag)]
        ov.join()
        res += [(a.cpu().numpy(), s.cpu().numpy()) for a, s in dev]
        # the drop-in call on this rank's HOST shard (bits packed on the CPU)
        from paper_2312_05385_b200.distributed import eval_thresholds_host_sharded, shard_range
        from paper_2312_05385_b200.engine import WindowEvaluator

        evf = WindowEvaluator.from_arrays(arrays, sites, prof, mode="hist")
        lo, hi = shard_range(arrays.n, rank, world)
        res.append(eval_thresholds_host_sharded(
            np.ascontiguousarray(arrays.errs[lo:hi]), arrays.correct[lo:hi].astype(np.float64),
            evf.serve, evf.vanilla_ms, diag, n_total=arrays.n))
        # two windows per rank, one all-reduce for both
        from paper_2312_05385_b200.distributed import evaluate_windows

        other = synth.config4_window(60_001, seed=7)
        sw2 = ShardedSweep(other, sites, prof, rank=rank, world=world)
        wa, ws = evaluate_windows([sw, sw2], rnd)
        res += [(wa[0], ws[0]), (wa[1], ws[1])]
        # the persistent multi-window sweep over this rank's shards, one all-reduce
        from paper_2312_05385_b200.distributed import WindowStream

        wsr = WindowStream([sw, sw2], order=[0, 1, 1, 0])
        da, dsv = wsr.run(diag)
        da, dsv = da.cpu().numpy(), dsv.cpu().numpy()
        res += [(da[q], dsv[q]) for q in range(4)]
        q.put((rank, [(a.tolist(), s.tolist()) for a, s in res]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sweep_matches_one_gpu(cuda):
    import torch.multiprocessing as mp

    from paper_2312_05385_b200 import synth
    from paper_2312_05385_b200.distributed import ShardedSweep
    from paper_2312_05385_b200.graph import find_feasible_sites

    prof = synth.config4_profile()
    sites = find_feasible_sites(prof)
    arrays = synth.config4_window(60_001)
    diag = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
    rnd = (np.arange(64) / 63.0)[np.random.default_rng(3).integers(0, 64, size=(50, 12))]
    one = [ShardedSweep(arrays, sites, prof).evaluate_many(th) for th in (diag, rnd)]
    one += one + one[:1]  # the overlapped exchange: diag, rnd, diag
    one += one[:1]  # host shards through eval_thresholds_host_sharded: diag
    other = synth.config4_window(60_001, seed=7)
    one += [one[1], ShardedSweep(other, sites, prof).evaluate_many(rnd)]  # evaluate_windows
    d_other = ShardedSweep(other, sites, prof).evaluate_many(diag)
    one += [one[0], d_other, d_other, one[0]]  # WindowStream order 0, 1, 1, 0 (diagonal rows)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank in (0, 1):
        for (acc, sav), (a1, s1) in zip(got[rank], one):
            assert np.array_equal(np.array(acc), a1)
            assert np.array_equal(np.array(sav), s1)


def _replica_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.update(WORLD_SIZE=str(world), RANK=str(rank), LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_05385_b200.replicas import run_replicas, serve

        agg = run_replicas("c1", n_batches=6)
        q.put((rank, agg))
    finally:
        dist.destroy_process_group()


def test_two_replica_serving_path(cuda):
    """Data-parallel serving: two replicas (both on cuda:0, gloo
    standing in for NCCL) each serve their round-robin share of 6 request batches
    through the captured EE graph with pinned H2D / D2H; rank 0 aggregates."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert got[1] is None
    agg = got[0]
    assert agg["replicas"] == 2 and agg["samples"] == 6 * 32
    assert agg["samples_per_s"] > 0 and agg["p50_batch_ms"] > 0
    assert 0.0 < agg["exit_rate"] <= 1.0
