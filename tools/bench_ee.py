"""EE batch inference throughput and latency (BASELINE configs 1-3).

For each config: thresholds from per-ramp err quantiles of a calibration
batch, then timed batches (CUDA events) in feedback mode (Apparate:
every input runs to completion, results released early) and compaction mode.
Reports samples/s, p50 batch latency, p50 per-request release latency, exit
rate, and the same model without ramps (vanilla, eager and as one CUDA graph)
for context. Backbones run in bf16 (see DTYPE_NOTE); ramp heads take the bf16
activations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2312_05385_b200 import ee_infer


def quantile_thresholds(pipe, x, q=(0.05, 0.10, 0.15, 0.20, 0.25, 0.30)):
    probe = pipe.run(x, [0.0] * pipe.n_ramps)
    err = probe.ramp_err.float().cpu().numpy()
    qs = list(q) + [q[-1]] * max(0, pipe.n_ramps - len(q))
    return [float(np.nanquantile(err[j], qs[j])) for j in range(pipe.n_ramps)]


def bench(name, pipe, make_input, batch, iters, warmup=5):
    th = quantile_thresholds(pipe, make_input(max(batch, 64)))
    out = {"config": name, "batch": batch, "ramps": pipe.n_ramps}
    for mode in ("feedback", "compact"):
        x = make_input(batch)
        for _ in range(warmup):
            pipe.run(x, th, mode=mode)
        lat, rel, exits = [], [], []
        for _ in range(iters):
            res = pipe.run(x, th, mode=mode, timed=True)
            lat.append(res.batch_ms)
            rel.extend(res.release_ms.tolist())
            exits.append(float((res.released_site.cpu().numpy() < pipe.n_ramps).mean()))
        out[mode] = {"samples_per_s": batch / (np.mean(lat) / 1e3),
                     "p50_batch_ms": float(np.percentile(lat, 50)),
                     "p50_request_release_ms": float(np.percentile(rel, 50)),
                     "exit_rate": float(np.mean(exits))}
    # feedback mode captured as one CUDA graph (thresholds in device memory)
    x = make_input(batch)
    runner = pipe.capture(x, th)
    for _ in range(warmup):
        runner.run()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        ev0.record()
        runner.run()
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ref = pipe.run(x, th)
    same = bool(torch.equal(runner.out.released_site, ref.released_site)
                and torch.equal(runner.out.released_label, ref.released_label))
    out["feedback_graph"] = {"samples_per_s": batch / (np.mean(ts) / 1e3),
                             "p50_batch_ms": float(np.percentile(ts, 50)),
                             "matches_eager": same, "ramps": "side stream, overlapped with the backbone"}
    # the same graph with the ramp heads serialised on the backbone's stream
    pipe.overlap_ramps = False
    try:
        srun = pipe.capture(x, th)
    finally:
        pipe.overlap_ramps = True
    for _ in range(warmup):
        srun.run()
    ts = []
    for _ in range(iters):
        ev0.record()
        srun.run()
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    out["feedback_graph_serial_ramps"] = {"samples_per_s": batch / (np.mean(ts) / 1e3),
                                          "p50_batch_ms": float(np.percentile(ts, 50))}
    # compaction mode as per-(segment, bucket) CUDA graphs (survivors gathered on the device)
    crun = pipe.capture_compact(x, th)
    for _ in range(warmup):
        crun.run()
    ts, exits = [], []
    for _ in range(iters):
        ev0.record()
        crun.run()
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
        exits.append(float((crun.out.released_site < pipe.n_ramps).float().mean().item()))
    # the same compaction scheduled on the device: one graph launch per batch
    # (SWITCH nodes pick each segment's bucket from the live count, no lag)
    for _ in range(warmup):
        crun.run_device()
    tsd = []
    for _ in range(iters):
        ev0.record()
        crun.run_device()
        ev1.record()
        ev1.synchronize()
        tsd.append(ev0.elapsed_time(ev1))
    fb = pipe.run(x, th)
    margin = 2e-3
    e = fb.ramp_err.float()
    near = torch.zeros(batch, dtype=torch.bool, device="cuda")
    for j, t in enumerate(th):
        near |= (e[j] - t).abs() < margin
    agree = bool(torch.equal(crun.out.released_site[~near], fb.released_site[~near]))
    out["compact_graph"] = {"samples_per_s": batch / (np.mean(ts) / 1e3),
                            "p50_batch_ms": float(np.percentile(ts, 50)),
                            "exit_rate": float(np.mean(exits)),
                            "graphs_captured": len(crun.graphs),
                            "matches_feedback_off_margin": agree,
                            "rows_within_margin": int(near.sum().item())}
    dsite = crun.run_device().released_site
    out["compact_device_graph"] = {"samples_per_s": batch / (np.mean(tsd) / 1e3),
                                   "p50_batch_ms": float(np.percentile(tsd, 50)),
                                   "matches_feedback_off_margin": bool(torch.equal(dsite[~near], fb.released_site[~near])),
                                   "schedule": "one graph launch: SWITCH nodes choose each segment's bucket on the device"}
    # vanilla: the same stages, no ramps
    x = make_input(batch)
    with torch.no_grad():
        for _ in range(warmup):
            h = x
            for s in pipe.stages:
                h = s(h)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(iters):
            ev0.record()
            h = x
            for s in pipe.stages:
                h = s(h)
            ev1.record()
            ev1.synchronize()
            ts.append(ev0.elapsed_time(ev1))
    out["vanilla"] = {"samples_per_s": batch / (np.mean(ts) / 1e3), "p50_batch_ms": float(np.percentile(ts, 50))}
    # vanilla captured as one CUDA graph too (the fair partner of feedback_graph)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.no_grad(), torch.cuda.stream(s):
        for _ in range(2):
            h = x
            for st in pipe.stages:
                h = st(h)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.no_grad(), torch.cuda.graph(g):
        h = x
        for st in pipe.stages:
            h = st(h)
    ts = []
    for _ in range(warmup):
        g.replay()
    for _ in range(iters):
        ev0.record()
        g.replay()
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    out["vanilla_graph"] = {"samples_per_s": batch / (np.mean(ts) / 1e3),
                            "p50_batch_ms": float(np.percentile(ts, 50))}
    out["dtype"] = DTYPE_NOTE
    return out


# Backbones in bf16 weights and activations (ResNets channels_last, the layout
# cuDNN's tensor-core convolutions want); EE_BENCH_AUTOCAST=1 restores the
# earlier fp32-weights + bf16-autocast setup for comparison.
AUTOCAST = os.environ.get("EE_BENCH_AUTOCAST") == "1"
DTYPE_NOTE = ("bf16 autocast over fp32 weights" if AUTOCAST
              else "bf16 weights/activations; CNNs channels_last with BatchNorm folded into the convolutions")


def _native_bf16(model, channels_last):
    if AUTOCAST:
        return
    ee_infer.prepare_bf16(model, channels_last)


def _image(g, channels_last):
    def make(b, shape):
        x = torch.randn(b, *shape, generator=g, device="cuda")
        if AUTOCAST:
            return x
        return x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last if channels_last
                                               else torch.contiguous_format)
    return make


def main():
    import contextlib

    torch.backends.cudnn.benchmark = True
    which = sys.argv[1:] or ["1", "2", "3"]
    g = torch.Generator(device="cuda").manual_seed(0)
    img = _image(g, True)
    res = []
    ctx = torch.autocast("cuda", dtype=torch.bfloat16) if AUTOCAST else contextlib.nullcontext()
    with ctx:
        if "1" in which:
            pipe, m = ee_infer.resnet18_cifar()
            _native_bf16(m, True)
            res.append(bench("resnet18_cifar_6ramps", pipe, lambda b: img(b, (3, 32, 32)), 32, 50))
        if "2" in which:
            pipe, m = ee_infer.bert_base()
            _native_bf16(m, False)
            res.append(bench("bert_base_12ramps_seq128_entropy", pipe,
                             lambda b: torch.randint(0, 30522, (b, 128), generator=g, device="cuda"), 64, 20))
        if "3" in which:
            pipe, m = ee_infer.resnet50_imagenet()
            _native_bf16(m, True)
            res.append(bench("resnet50_imagenet_16ramps", pipe, lambda b: img(b, (3, 224, 224)), 256, 10))
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
