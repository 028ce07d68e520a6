"""Closed-loop early-exit serving on the GPU (the kept control
loop of pkg/src/eesim/serving.py driven by the on-GPU exit controller).

The reference's `serving.run` (serving.py:176-359) replays logged ramp signals
through a latency profile. Here the same loop serves real request batches
through an EEPipeline (ee_infer.py) on the GPU:

  * batches form exactly as in serving.py:218-223 (work-conserving: at
    start = max(free_at, next arrival), take every arrived request up to
    max_batch), but a batch's busy time is the MEASURED GPU time of the
    pipeline, and each request's release time is its exit ramp's CUDA event;
  * every ramp runs in feedback mode (Apparate semantics): all
    inputs run to completion, results leave at the first ramp whose error is
    strictly below its threshold (engine.py:207), and every ramp's (err,
    label) plus the final label are observed for every request;
  * responses feed the controller in release order (serving.py:260): the
    accuracy monitor (tuner.py:56-81) sees whether the released label matches
    the final model's, the request joins the bounded tuning history
    (serving.py:278-280), and when should_trigger fires, Algorithm 1
    (tuner.tune, on the GPU) retunes the thresholds. The new thresholds are
    written into the device tensor the exit controllers read, so the next
    batch uses them with no re-capture.

`LiveReport.batches` keeps, per batch, the thresholds it ran with and each
request's RequestRecord, so tests can replay every decision through the
reference exit rule and every retune through the pinned oracle tuner.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.engine import EEConfig, WindowEvaluator
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.graph import ModelProfile, find_feasible_sites
from paper_2312_05385_b200.trace import RampSignal, RequestRecord, WindowArrays
from paper_2312_05385_b200.tuner import AccuracyMonitor, TunerParams, should_trigger, tune


@dataclass
class LiveParams:
    max_batch: int = 32
    acc_constraint: float = 0.99
    tuner: TunerParams = field(default_factory=TunerParams)


@dataclass
class LiveRow:
    id: int
    arrival_ms: float
    queue_ms: float
    serve_ms: float
    total_ms: float
    exit_site: str | None
    correct: bool
    batch: int


@dataclass
class LiveBatch:
    start_ms: float
    busy_ms: float
    thresholds: tuple[float, ...]
    records: list  # RequestRecord per request (ramp signals + final label)
    released_site: np.ndarray  # ramp index or n_ramps


@dataclass
class LiveReport:
    rows: list[LiveRow]
    batches: list[LiveBatch]
    tunes: list[dict]
    accuracy: float
    p50_ms: float
    throughput_rps: float


def _stage_times(pipe, x, repeats: int):
    torch = nat.torch_cuda()
    stage_ms = np.zeros(len(pipe.stages))
    ramp_ms = np.zeros(len(pipe.stages))
    with torch.no_grad():
        for _ in range(repeats):
            h = x
            for j, stage in enumerate(pipe.stages):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h2 = stage(h)
                e1.record()
                e1.synchronize()
                stage_ms[j] += e0.elapsed_time(e1) / repeats
                head = pipe.ramps.get(j)
                if head is not None:
                    e0.record()
                    head(h2, 2.0)
                    e1.record()
                    e1.synchronize()
                    ramp_ms[j] += e0.elapsed_time(e1) / repeats
                h = h2
    return stage_ms, ramp_ms


def profile_pipeline(pipe, example, *, repeats: int = 5) -> ModelProfile:
    """A chain ModelProfile of the pipeline's stages with measured per-stage and
    per-ramp GPU milliseconds at batch 1 and at the example's batch size (the
    tuner's serve table, engine.py:124-132, is taken at batch 1 as in
    serving.py:286). Node "st{j}" is the cut after stage j, so the feasible
    site of the ramp at stage j is "st{j}"."""
    b = int(example.shape[0])
    s1, r1 = _stage_times(pipe, example[:1], repeats)
    sb, rb = _stage_times(pipe, example, repeats) if b > 1 else (s1, r1)
    nodes = [f"st{j}" for j in range(len(pipe.stages))]
    batches = sorted({1, b})

    def table(x1, xb):
        return {bb: float(x1 if bb == 1 else max(xb, x1)) for bb in batches}  # monotone in batch

    lat = {n: table(s1[j], sb[j]) for j, n in enumerate(nodes)}
    ramp = {n: table(r1[j], rb[j]) for j, n in enumerate(nodes[:-1])}
    return ModelProfile(nodes, list(zip(nodes, nodes[1:])), lat, ramp, nodes[-1], name="live")


def _graph_runner(pipe, bsz: int, example, thresholds):
    """The pipeline's timed feedback-mode graph for batch size `bsz`, captured on
    first use and kept on the pipeline (one graph per batch size the server forms)."""
    cache = pipe.__dict__.setdefault("_live_graphs", {})
    key = (bsz, tuple(example.shape[1:]), example.dtype, example.stride()[1:])
    run = cache.get(key)
    if run is None:
        run = pipe.capture(example[:bsz], thresholds, timed=True)
        run.version = None
        cache[key] = run
    return run


def serve_live(pipe, requests, arrivals_ms, profile: ModelProfile, thresholds, params: LiveParams,
               *, tune_on_trigger: bool = True, graphs: bool = False) -> LiveReport:
    """Serve `requests` [n, ...] (CUDA tensor) arriving at `arrivals_ms` (sorted).

    graphs: every batch is one replay of a CUDA graph captured per batch size
    (EEPipeline.capture(timed=True)): busy time and per-ramp release times come
    from event nodes inside the graph, so a batch costs its GPU time instead of
    the eager pipeline's per-kernel launch overhead. Decisions are the same
    kernels on the same thresholds (a retune is copied into every graph's
    device threshold vector before its next replay)."""
    torch = nat.torch_cuda()
    n = int(requests.shape[0])
    arrivals_ms = np.asarray(arrivals_ms, dtype=np.float64)
    if n == 0:
        return LiveReport([], [], [], 1.0, 0.0, 0.0)
    if len(arrivals_ms) != n or np.any(np.diff(arrivals_ms) < 0):
        raise ParameterError("arrivals must be sorted, one per request")
    all_sites = {s.position: s for s in find_feasible_sites(profile)}
    sites = [all_sites[f"st{j}"] for j in pipe.ramp_order]
    R = len(sites)
    th_dev = torch.tensor([float(t) for t in thresholds], dtype=torch.float64, device="cuda")
    config = EEConfig(tuple(zip(sites, [float(t) for t in thresholds])))
    monitor = AccuracyMonitor(params.tuner.accuracy_window)
    history: list[RequestRecord] = []
    # the history's columns, kept as a ring in step with `history` (same rows,
    # same order), so a retune builds its device window from arrays instead of
    # re-packing every RequestRecord (trace.window_arrays: ~0.8 ms per 1,000)
    cap = max(1, params.tuner.tuning_history)
    ring_err = np.empty((cap, R))
    ring_ok = np.ones((cap, R + 1), dtype=np.uint8)
    ring_start = 0
    rows: list[LiveRow] = []
    batches: list[LiveBatch] = []
    tunes: list[dict] = []
    version = 0  # bumped by every retune; a graph copies the thresholds when behind
    i = 0
    free_at = float(arrivals_ms[0])
    first = float(arrivals_ms[0])
    last_end = first
    while i < n:
        start = max(free_at, float(arrivals_ms[i]))
        j = i
        while j < n and j - i < params.max_batch and arrivals_ms[j] <= start:
            j += 1
        if graphs:
            run = _graph_runner(pipe, j - i, requests, config.thresholds)
            if run.version != version:
                run.th.copy_(th_dev)
                run.version = version
            res = run.run(requests[i:j])
        else:
            res = pipe.run(requests[i:j], th_dev, mode="feedback", timed=True)
        busy = float(res.batch_ms)
        err = res.ramp_err.double().cpu().numpy()
        lab = res.ramp_label.cpu().numpy()
        fin = res.final_label.cpu().numpy()
        rel_site = res.released_site.cpu().numpy()
        rel_label = res.released_label.cpu().numpy()
        recs = []
        served = []
        ok = (lab == fin[None, :]).T  # [batch, R] released label at ramp r == final label
        for q in range(j - i):
            rid = i + q
            sig = {sites[r].position: RampSignal(float(err[r, q]), int(lab[r, q])) for r in range(R)}
            rec = RequestRecord(rid, float(arrivals_ms[rid]), sig, int(fin[q]))
            recs.append(rec)
            site = int(rel_site[q])
            correct = bool(rel_label[q] == fin[q])
            served.append((start + float(res.release_ms[q]), rid, rec, site, correct, q))
        batches.append(LiveBatch(start, busy, tuple(config.thresholds), recs, rel_site.copy()))
        served.sort(key=lambda t: (t[0], t[1]))  # release order feeds the monitor (serving.py:260)
        free_at = start + busy
        last_end = free_at
        for release, rid, rec, site, correct, q in served:
            queue = start - rec.arrival_ms
            rows.append(LiveRow(rid, rec.arrival_ms, queue, release - start, release - rec.arrival_ms,
                                sites[site].position if site < R else None, correct, j - i))
            monitor.push(correct)
            history.append(rec)
            slot = (ring_start + len(history) - 1) % cap
            ring_err[slot] = err[:, q]
            ring_ok[slot, :R] = ok[q]
            if len(history) > params.tuner.tuning_history:
                history.pop(0)
                ring_start = (ring_start + 1) % cap
            if tune_on_trigger and R and should_trigger(monitor, params.acc_constraint):
                n_h = len(history)
                order = (ring_start + np.arange(n_h)) % cap  # oldest first, as `history`
                ev = WindowEvaluator.from_arrays(
                    WindowArrays(ring_err[order], ring_ok[order]), sites, profile, batch=1,
                    records=history)
                res_t = tune(history, sites, params.tuner, profile, evaluator=ev)
                new = res_t.threshold_vector(sites)
                tunes.append({"after_request": rid, "history": list(history),
                              "thresholds": new, "savings_ms": res_t.savings_ms,
                              "accuracy": res_t.accuracy})
                config = config.with_thresholds(new)
                th_dev.copy_(th_dev.new_tensor(new))
                version += 1
        i = j
    bits = [r.correct for r in rows]
    makespan = last_end - first
    return LiveReport(
        rows, batches, tunes,
        accuracy=float(np.mean(bits)),
        p50_ms=float(np.percentile([r.total_ms for r in rows], 50)),  # linear, manifest.py:100-107
        throughput_rps=len(rows) / (makespan / 1000.0) if makespan > 0 else 0.0,
    )
