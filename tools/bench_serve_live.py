"""Closed-loop EE serving of ResNet-18 CIFAR on the GPU (serve_live.py): Poisson
arrivals, work-conserving batching (max 32), monitor-triggered GPU retuning.
Prints one JSON line: p50 latency, throughput, accuracy vs the final model,
exit rate, retunes and their mean GPU time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import ee_infer
from paper_2312_05385_b200.serve_live import LiveParams, profile_pipeline, serve_live
from paper_2312_05385_b200.tuner import TunerParams

torch.backends.cudnn.benchmark = True  # every batch shape 1..32 is autotuned in the warm-up below
pipe, m = ee_infer.resnet18_cifar()
# same backbone form as tools/bench_ee.py: BatchNorm folded, bf16, channels_last,
# the blocks on the repo's kernels
ee_infer.prepare_bf16(m, True)
n = int(os.environ.get("N", 2048))
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(n, 3, 32, 32, generator=g, device="cuda").to(torch.bfloat16).contiguous(
    memory_format=torch.channels_last)
for bsz in range(1, 33):  # warm every batch shape the server can form (cuDNN picks its kernels once)
    for _ in range(2):
        pipe.run(x[:bsz], [0.0] * pipe.n_ramps)
torch.cuda.synchronize()
prof = profile_pipeline(pipe, x[:32])
probe = pipe.run(x[:256], [0.0] * pipe.n_ramps)
err = probe.ramp_err.float().cpu().numpy()
th0 = [float(np.quantile(err[j], 0.2)) for j in range(pipe.n_ramps)]
rate = float(os.environ.get("RATE_PER_MS", 8.0))
arr = np.cumsum(np.random.default_rng(1).exponential(1.0 / rate, size=n))
params = LiveParams(max_batch=32, acc_constraint=0.95, tuner=TunerParams(acc_loss_budget=0.02))
serve_live(pipe, x[:256], arr[:256], prof, th0, params)  # warm
t0 = time.perf_counter()
eager = serve_live(pipe, x, arr, prof, th0, params)
wall_eager = time.perf_counter() - t0
# every batch as one replay of a graph captured per batch size (captured here,
# outside the measured loop, for every size 1..32 the server can form)
for bsz in range(1, 33):
    serve_live(pipe, x[:bsz], np.zeros(bsz), prof, th0, params, tune_on_trigger=False, graphs=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = serve_live(pipe, x, arr, prof, th0, params, graphs=True)
wall = time.perf_counter() - t0
vanilla_ms = prof.model_latency(32)
print(json.dumps({
    "config": f"config1 closed loop: ResNet-18 CIFAR 6 ramps (bf16, channels_last, BN folded), {n} requests, "
              f"Poisson {rate}/ms, max batch 32",
    "p50_ms": rep.p50_ms, "throughput_rps": rep.throughput_rps, "accuracy_vs_final": rep.accuracy,
    "exit_rate": float(np.mean([r.exit_site is not None for r in rep.rows])),
    "batches": len(rep.batches), "retunes": len(rep.tunes),
    "vanilla_batch32_ms_profile": vanilla_ms, "host_wall_s": wall,
    "batches_as": "one CUDA graph replay per batch (captured per batch size; busy and release times from "
                  "event nodes in the graph)",
    "mean_batch_ms": float(np.mean([b.busy_ms for b in rep.batches])),
    "eager": {"p50_ms": eager.p50_ms, "throughput_rps": eager.throughput_rps, "batches": len(eager.batches),
              "retunes": len(eager.tunes), "mean_batch_ms": float(np.mean([b.busy_ms for b in eager.batches])),
              "host_wall_s": wall_eager, "batches_as": "eager pipeline, CUDA events per ramp"}}))
