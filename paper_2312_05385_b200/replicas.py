"""Data-parallel EE serving: one model replica and one exit controller per GPU
(SURVEY §8e "Serving (C1-C3, C5): replicas only"; the paper runs "a separate
controller per model replica"; the per-replica
serving loop is pkg/src/eesim/serving.py:176-359).

One process per GPU (torchrun). The request stream is cut into batches of the
config's batch size; replica g serves batches g, g + W, g + 2W, ... (no
collective on the data path — requests are independent). Each replica replays
its feedback-mode EE pipeline as one CUDA graph (ee_infer.GraphRunner): every
batch's input is copied host→device from pinned memory, the whole backbone plus
every ramp head / fused exit controller runs, and the released (label, site)
of every request is copied back. Per-batch latency is CUDA-event timed on the
replica's stream; the job's throughput is all requests ÷ the slowest replica's
device time, and p50 is over the batch latencies of every replica
(np.percentile linear, as manifest.py:100-107).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2312_05385_b200.errors import ParameterError

CONFIGS = {
    "c1": ("resnet18_cifar_6ramps", 32),
    "c2": ("bert_base_12ramps_seq128_entropy", 64),
    "c3": ("resnet50_imagenet_16ramps", 256),
}


def replica_batches(n_batches: int, rank: int, world: int) -> list[int]:
    """Global batch indices served by replica `rank` (round-robin dispatch)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank {rank} for world size {world}")
    if n_batches < 0:
        raise ParameterError("n_batches must be >= 0")
    return list(range(rank, n_batches, world))


@dataclass
class ReplicaStats:
    rank: int
    samples: int
    device_ms: float                 # this replica's timed region (CUDA events)
    batch_ms: list = field(default_factory=list)
    exits: int = 0
    near_ties: int = 0


def aggregate(stats: ReplicaStats, group=None) -> dict:
    """Whole-job numbers from every replica's stats (gathered over
    torch.distributed when initialised; a single replica otherwise)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        allst = [None] * dist.get_world_size(group)
        dist.all_gather_object(allst, stats, group=group)
    else:
        allst = [stats]
    samples = sum(s.samples for s in allst)
    t_max = max(s.device_ms for s in allst)
    lat = [x for s in allst for x in s.batch_ms]
    return {
        "replicas": len(allst),
        "samples": samples,
        "samples_per_s": samples / (t_max / 1e3) if t_max > 0 else None,
        "p50_batch_ms": float(np.percentile(lat, 50)) if lat else None,
        "p90_batch_ms": float(np.percentile(lat, 90)) if lat else None,
        "slowest_replica_ms": t_max,
        "per_replica_samples_per_s": [s.samples / (s.device_ms / 1e3) if s.device_ms else None
                                      for s in allst],
        "exit_rate": sum(s.exits for s in allst) / samples if samples else None,
        "near_tie_rows": sum(s.near_ties for s in allst),
    }


def build_pipeline(config: str):
    """(pipeline, input maker(b, generator) -> CUDA tensor, batch) in serving form:
    bf16 weights/activations, CNNs channels_last with BatchNorm folded."""
    import torch

    from paper_2312_05385_b200 import ee_infer

    if config not in CONFIGS:
        raise ParameterError(f"unknown serving config {config!r} ({sorted(CONFIGS)})")
    batch = CONFIGS[config][1]
    if config == "c1":
        pipe, m = ee_infer.resnet18_cifar()
        ee_infer.prepare_bf16(m, channels_last=True)
        shape = (3, 32, 32)
    elif config == "c3":
        pipe, m = ee_infer.resnet50_imagenet()
        ee_infer.prepare_bf16(m, channels_last=True)
        shape = (3, 224, 224)
    else:
        pipe, m = ee_infer.bert_base()
        ee_infer.prepare_bf16(m, channels_last=False)

        def tokens(b, g):
            return torch.randint(0, 30522, (b, 128), generator=g, device="cuda")
        return pipe, tokens, batch

    def images(b, g):
        x = torch.randn(b, *shape, generator=g, device="cuda")
        return x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    return pipe, images, batch


def serve(config: str, n_batches: int, rank: int, world: int, *, warmup: int = 3,
          q=(0.05, 0.10, 0.15, 0.20, 0.25, 0.30)) -> ReplicaStats:
    """Serve this replica's share of `n_batches` request batches (synthetic inputs,
    seeded by global batch index, staged in pinned host memory) and return its stats.
    Thresholds: per-ramp err quantiles of a calibration batch (identical on every
    replica: same seed)."""
    import torch

    pipe, make, batch = build_pipeline(config)
    g = torch.Generator(device="cuda").manual_seed(12345)
    probe = pipe.run(make(batch, g), [0.0] * pipe.n_ramps)
    err = probe.ramp_err.double().cpu().numpy()
    qs = list(q) + [q[-1]] * max(0, pipe.n_ramps - len(q))
    th = [float(np.nanquantile(err[j], qs[j])) for j in range(pipe.n_ramps)]
    mine = replica_batches(n_batches, rank, world)
    # request batches live in pinned host memory (the serving front end's buffers)
    host = []
    for i in mine:
        gi = torch.Generator(device="cuda").manual_seed(1000 + i)
        host.append(make(batch, gi).cpu().pin_memory())
    runner = pipe.capture(make(batch, g), th)
    out_host = torch.empty((2, batch), dtype=torch.int32).pin_memory()
    for i in range(min(warmup, len(host))):
        runner.x.copy_(host[i], non_blocking=True)
        runner.run()
    torch.cuda.synchronize()
    stats = ReplicaStats(rank, batch * len(mine), 0.0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in mine]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    start.record()
    for k, xh in enumerate(host):
        ev[k][0].record()
        runner.x.copy_(xh, non_blocking=True)
        res = runner.run()
        out_host[0].copy_(res.released_label, non_blocking=True)
        out_host[1].copy_(res.released_site, non_blocking=True)
        ev[k][1].record()
    end.record()
    torch.cuda.synchronize()
    stats.device_ms = start.elapsed_time(end) if host else 0.0
    stats.batch_ms = [a.elapsed_time(b) for a, b in ev]
    # exit and near-tie counts (untimed second pass: the graph's outputs are reused)
    for xh in host:
        runner.x.copy_(xh, non_blocking=True)
        res = runner.run()
        stats.exits += int((res.released_site < pipe.n_ramps).sum().item())
        stats.near_ties += res.near_tie_count()
    return stats


def run_replicas(config: str = "c3", n_batches: int | None = None) -> dict | None:
    """Entry point under torchrun (one process per GPU) or a single process.
    Returns the aggregate on rank 0 (None elsewhere)."""
    import os

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if n_batches is None:
        n_batches = 8 * world
    st = serve(config, n_batches, rank, world)
    agg = aggregate(st)
    agg.update({"config": CONFIGS[config][0], "batch_per_replica": CONFIGS[config][1],
                "batches": n_batches, "n_gpus": world,
                "how": "one replica + controller per GPU, round-robin request batches, "
                       "pinned H2D of each batch + D2H of released (label, site) inside the "
                       "timed region, feedback-mode EE graph; samples / slowest replica's "
                       "CUDA-event time"})
    return agg if rank == 0 else None
