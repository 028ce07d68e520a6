"""Early-exit batch inference on the GPU (BASELINE configs 1-3; north star (1)-(2)).

A backbone is split into stages at its ramp sites. After each active site the
ramp head + exit controller (heads.py) pools, classifies, scores confidence,
compares against the site's threshold, clears the exiting rows from the alive
mask in place and scatters their (label, err, site) to their request slots —
one launch per ramp, no host round trip in feedback mode.

Two modes, SURVEY §7 hard part 6:
  * "feedback" (default; Apparate semantics): results exit early
    but every input runs to completion, so every active ramp's (err, label)
    and the final label are observed for all inputs — exactly the signals
    the accuracy monitor and the threshold tuner consume (serving.py:277-281).
  * "compact": surviving rows are gathered into a dense batch after each ramp
    (stable ascending order), so later stages run only on non-exited rows;
    later ramps' signals of exited rows are then censored (NaN / -1).

The exit rule is the reference's (engine.py:189-220): first active ramp with
err strictly below its threshold; otherwise the final model label is
released. `BatchResult.records()` re-expresses a batch as RequestRecords, the
form the reference's tuner consumes.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.convnet import can_run_into, run_into
from paper_2312_05385_b200.heads import (ExitController, LargeRampHead, SlotTable, compact_fill, compact_meta,
                                        compact_rows, exit_from_logits, gemm, scatter_signals)

# North star: a sample whose confidence lies within 1e-5 of a threshold is a
# near-tie — its exit decision may legitimately differ from an fp64 CPU oracle,
# so it is reported rather than counted as a mismatch.
NEAR_TIE_EPS = 1e-5


@dataclass
class BatchResult:
    released_label: "object"  # i32 [B]
    released_site: "object"   # i32 [B]: ramp index, or n_ramps for the final model
    released_err: "object"    # f32 [B]
    ramp_err: "object"        # f32 [R, B] every active ramp's error score (NaN if censored)
    ramp_label: "object"      # i32 [R, B]
    final_label: "object"     # i32 [B] (-1 if censored in compaction mode)
    release_ms: np.ndarray | None = None  # per request, from batch start (host, if timed)
    batch_ms: float | None = None
    thresholds: "object" = None  # the thresholds this batch was decided under (host list or CUDA f64 [R])
    events: "object" = None  # (start, per-ramp marks, end) CUDA events of a graph-captured timed batch

    def near_ties(self, thresholds=None, eps: float = NEAR_TIE_EPS):
        """bool [B] (CUDA): rows with |err_j - t_j| < eps at some active ramp j the
        row reached (j <= its release site) — the decisions the north star
        reports instead of requiring them to match an fp64 oracle bit for bit
        (the strict rule is engine.py:207). NaN (censored) entries never tie."""
        import torch

        th = self.thresholds if thresholds is None else thresholds
        if th is None:
            raise ParameterError("near_ties needs the thresholds the batch ran under")
        r, b = self.ramp_err.shape
        if r == 0:
            return torch.zeros(b, dtype=torch.bool, device=self.ramp_err.device)
        if not hasattr(th, "data_ptr"):
            th = torch.tensor([float(t) for t in th], dtype=torch.float64)
        th = th.to(self.ramp_err.device, torch.float64).view(r, 1)
        close = (self.ramp_err.double() - th).abs() < eps
        reached = torch.arange(r, device=self.ramp_err.device).view(r, 1) <= \
            self.released_site.view(1, b).long()
        return (close & reached).any(dim=0)

    def near_tie_count(self, thresholds=None, eps: float = NEAR_TIE_EPS) -> int:
        return int(self.near_ties(thresholds, eps).sum().item())

    def records(self, site_names: Sequence[str], first_id: int = 0, arrival_ms: float = 0.0):
        """The batch as reference RequestRecords (err/label per site, final label)."""
        from paper_2312_05385_b200.trace import RampSignal, RequestRecord

        err = self.ramp_err.double().cpu().numpy()
        lab = self.ramp_label.cpu().numpy()
        fin = self.final_label.cpu().numpy()
        out = []
        for i in range(err.shape[1]):
            sig = {name: RampSignal(float(err[j, i]), int(lab[j, i])) for j, name in enumerate(site_names)}
            out.append(RequestRecord(first_id + i, arrival_ms, sig, int(fin[i])))
        return out


@dataclass
class EEPipeline:
    """stages[j] maps the previous activation to site j's activation; the last
    stage produces final logits. ramps maps a stage index to its ramp head."""

    stages: list
    ramps: dict
    site_names: list = field(default_factory=list)
    # feedback mode: ramp heads run on a side stream, overlapped with the next
    # stages (they feed nothing downstream but each other, in ramp order)
    overlap_ramps: bool = True

    def __post_init__(self):
        self.ramp_order = sorted(self.ramps)
        if any(j >= len(self.stages) - 1 for j in self.ramp_order):
            raise ParameterError("ramps must sit before the final stage")
        if not self.site_names:
            self.site_names = [f"s{j}" for j in self.ramp_order]

    @property
    def n_ramps(self) -> int:
        return len(self.ramp_order)

    def capture(self, example, thresholds, *, timed: bool = False) -> "GraphRunner":
        """Capture one feedback-mode batch into a CUDA graph (static shapes; the
        thresholds live in device memory, so retuning needs no re-capture).
        timed: every replay fills batch_ms / release_ms from event nodes."""
        return GraphRunner(self, example, thresholds, timed=timed)

    def capture_compact(self, example, thresholds) -> "CompactRunner":
        """Compaction mode as CUDA graphs, one per (segment, batch bucket)."""
        return CompactRunner(self, example, thresholds)

    def run(self, x, thresholds, *, mode: str = "feedback",
            timed: bool = False) -> BatchResult:
        torch = nat.torch_cuda()
        if len(thresholds) != self.n_ramps:
            raise ParameterError(f"{self.n_ramps} thresholds expected")
        if mode not in ("feedback", "compact"):
            raise ParameterError("mode must be 'feedback' or 'compact'")
        b = x.shape[0]
        R = self.n_ramps
        dev = "cuda"
        # thresholds: host floats, or a CUDA f64 [R] tensor read by the kernels at run time
        dev_th = hasattr(thresholds, "data_ptr")
        th_record = thresholds if dev_th else [float(t) for t in thresholds]
        if dev_th:
            thresholds = [thresholds[r : r + 1] for r in range(R)]
        alive = torch.ones(b, dtype=torch.uint8, device=dev)
        # request slot of each live row (feedback mode: the identity, which the
        # kernels take as a null slot map)
        rows = torch.arange(b, dtype=torch.int32, device=dev) if mode == "compact" else None
        if mode == "feedback":
            # every row reaches every ramp (each writes err/label for all rows) and
            # is released exactly once (at a ramp or by the final model), so the
            # result tables need no fill kernels
            slots = SlotTable.uninitialized(b)
            ramp_err = torch.empty((R, b), dtype=torch.float32, device=dev)
            ramp_label = torch.empty((R, b), dtype=torch.int32, device=dev)
            final_label = torch.empty((b,), dtype=torch.int32, device=dev)
        else:
            slots = SlotTable.empty(b)
            ramp_err = torch.full((R, b), float("nan"), dtype=torch.float32, device=dev)
            ramp_label = torch.full((R, b), -1, dtype=torch.int32, device=dev)
            final_label = torch.full((b,), -1, dtype=torch.int32, device=dev)
        marks = []
        # timed="graph": inside a CUDA graph capture; the events become record
        # nodes (external) and GraphRunner reads them after each replay
        ext = timed == "graph"

        def event():
            return torch.cuda.Event(enable_timing=True, external=ext)

        if timed:
            start = event()
            start.record()
        main = torch.cuda.current_stream()
        side = None
        if mode == "feedback" and self.overlap_ramps and R:
            # The ramp heads form their own chain on a side stream (ramp j reads
            # the alive mask ramp j - 1 wrote), each forked off the main stream
            # right after its stage, so a head's pooling / FC / compare runs
            # while the backbone moves on; joined before the final classifier.
            # Stage outputs a head still reads are held until the join (the
            # caching allocator must not hand them to a later stage).
            side = self._side_stream(torch)
            side.wait_stream(main)
        held = []
        h = x
        r = 0
        with torch.no_grad():
            for j, stage in enumerate(self.stages[:-1]):
                if h.shape[0] == 0:
                    break
                h = stage(h)
                head = self.ramps.get(j)
                if head is None:
                    continue
                th = thresholds[r] if dev_th else float(thresholds[r])
                if side is not None:
                    side.wait_stream(main)
                    held.append(h)
                    with torch.cuda.stream(side):
                        head(h, th, alive=alive, slot=rows, slots=slots,
                             out_err=ramp_err[r], out_label=ramp_label[r], compact=False)
                        if timed:
                            ev = event()
                            ev.record()
                            marks.append(ev)
                    r += 1
                    continue
                if mode == "feedback":  # rows are the identity: write signals in place
                    res = head(h, th, alive=alive, slot=rows, slots=slots,
                               out_err=ramp_err[r], out_label=ramp_label[r], compact=False)
                else:
                    res = head(h, th, alive=alive, slot=rows, slots=slots)
                    scatter_signals(res.err, res.label, rows, ramp_err[r], ramp_label[r])
                if timed:
                    ev = event()
                    ev.record()
                    marks.append(ev)
                if mode == "compact":
                    n = int(res.n_keep.item())  # host sync: the next stage's batch size
                    # gather in the activation's own memory format (index_select
                    # would turn a channels_last map into NCHW for every later conv)
                    h = compact_rows(h, res.keep, res.n_keep)[:n]
                    rows = rows.index_select(0, res.keep[:n].long())
                    alive = torch.ones(n, dtype=torch.uint8, device=dev)
                r += 1
            if h.shape[0]:
                logits = self.stages[-1](h).float()
                if side is not None:  # join: every ramp has decided
                    main.wait_stream(side)
                    held.clear()
                # every still-alive row is released with the final model's label
                # (argmax, first maximum: torch.argmax's rule); feedback mode
                # takes every row's label straight from the kernel
                if mode == "feedback":
                    exit_from_logits(logits.contiguous(), 2.0, conf="maxprob", site=R, alive=alive,
                                     slots=slots, out_label=final_label, compact=False)
                else:
                    final_label.index_copy_(0, rows.long(), torch.argmax(logits, dim=1).to(torch.int32))
                    exit_from_logits(logits.contiguous(), 2.0, conf="maxprob", site=R, alive=alive,
                                     slot=rows, slots=slots, compact=True)
        if side is not None:
            main.wait_stream(side)
        out = BatchResult(slots.label, slots.site, slots.err, ramp_err, ramp_label, final_label,
                          thresholds=th_record)
        if timed == "graph":
            end = event()
            end.record()
            out.events = (start, marks, end)
        elif timed:
            end = event()
            end.record()
            end.synchronize()
            t = [start.elapsed_time(m) for m in marks] + [start.elapsed_time(end)]
            site = slots.site.cpu().numpy()
            out.release_ms = np.asarray(t)[np.clip(site, 0, R)]
            out.batch_ms = t[-1]
        return out


    def _side_stream(self, torch):
        s = self.__dict__.get("_side")
        if s is None or s.device != torch.device("cuda", torch.cuda.current_device()):
            s = torch.cuda.Stream()
            self.__dict__["_side"] = s
        return s


class GraphRunner:
    """A feedback-mode EEPipeline batch replayed as one CUDA graph: the whole
    backbone + every ramp head / exit controller + scatter in one launch from
    the host (the per-ramp Python and launch overhead disappears)."""

    def __init__(self, pipe: EEPipeline, example, thresholds, *, timed: bool = False):
        torch = nat.torch_cuda()
        self.pipe = pipe
        self.x = example.clone()
        self.th = torch.tensor([float(t) for t in thresholds], dtype=torch.float64, device="cuda")
        self.timed = timed
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):  # warm-up: grow workspaces, pick cuDNN algorithms
                pipe.run(self.x, self.th)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            # timed: the batch start, every ramp's decision and the end are event
            # record NODES of the graph (external events), so a replay is timed on
            # the device exactly like an eager timed run
            self.out = pipe.run(self.x, self.th, timed="graph" if timed else False)

    def set_thresholds(self, thresholds):
        self.th.copy_(self.th.new_tensor([float(t) for t in thresholds]))

    def run(self, x=None) -> BatchResult:
        if x is not None:
            self.x.copy_(x)
        self.graph.replay()
        if self.timed:
            start, marks, end = self.out.events
            end.synchronize()
            t = [start.elapsed_time(m) for m in marks] + [start.elapsed_time(end)]
            site = self.out.released_site.cpu().numpy()
            self.out.release_ms = np.asarray(t)[np.clip(site, 0, len(marks))]
            self.out.batch_ms = t[-1]
        return self.out


def compaction_segments(ramp_order, n_stages: int):
    """[(first stage, last stage)] of a compacted batch: each segment ends at a
    ramp site, the last one at the final classifier (stage n_stages - 1)."""
    ends = list(ramp_order) + [n_stages - 1]
    starts = [0] + [e + 1 for e in ends[:-1]]
    return list(zip(starts, ends))


def compaction_buckets(b: int):
    """Batch buckets of a compacted segment: multiples of B/16 and the powers of
    two below B/16 (every live count maps to the smallest bucket >= it)."""
    granule = max(1, b // 16)
    return sorted({min(b, 1 << k) for k in range(granule.bit_length() + 1)}
                  | set(range(granule, b + 1, granule)) | {b})


class CompactRunner:
    """Compaction mode (north star (2): downstream blocks run only on the rows
    that have not exited) without per-stage host work.

    The pipeline is cut into segments, each ending at a ramp (the last one at
    the final classifier). A segment runs at a batch bucket >= its live row
    count (a multiple of B/16, or a power of two below that), as a CUDA graph
    captured once per (segment, bucket):
    stages -> ramp head / exit controller (compaction on) -> scatter of the
    exiting rows -> gather of the survivors' activations, request slots and
    alive bytes into the next segment's fixed input buffers (ee_compact_rows /
    ee_compact_meta, all on the device). Rows past the live count inside a
    bucket are padding: alive = 0 and a dummy request slot (index B of the
    B + 1 result tables), so they never exit, scatter or count.

    Bucket choice never stalls the device: every segment's graph copies its
    survivor count into pinned host memory, and segment k + 1 is launched at
    the bucket of the count after segment k - 1 (an upper bound of its live
    rows: counts only fall), which the host reads while segment k runs. The
    host therefore stays one segment ahead and the GPU never drains between
    segments; the price is one segment of lag in shrinking. The run stops
    once a count reaches zero. Decisions equal EEPipeline.run's
    compaction mode (same kernels on the same rows), and rows far from a
    threshold equal feedback mode's."""

    def __init__(self, pipe: EEPipeline, example, thresholds):
        torch = nat.torch_cuda()
        self.pipe = pipe
        self.B = b = example.shape[0]
        self.R = R = pipe.n_ramps
        self.th = torch.tensor([float(t) for t in thresholds], dtype=torch.float64, device="cuda")
        self.segments = compaction_segments(pipe.ramp_order, len(pipe.stages))
        self.buckets = compaction_buckets(b)
        dev = "cuda"
        # result tables: B request slots + one dummy slot for padding rows
        self.slots = SlotTable(torch.empty(b + 1, dtype=torch.int32, device=dev),
                               torch.empty(b + 1, dtype=torch.float32, device=dev),
                               torch.empty(b + 1, dtype=torch.int32, device=dev))
        self.ramp_err = torch.empty((R, b + 1), dtype=torch.float32, device=dev)
        self.ramp_label = torch.empty((R, b + 1), dtype=torch.int32, device=dev)
        self.final_label = torch.empty((b + 1,), dtype=torch.int32, device=dev)
        self.n_live = torch.zeros(len(self.segments), dtype=torch.int32, device=dev)
        self.n_host = torch.zeros(len(self.segments), dtype=torch.int32, pin_memory=True)
        self.done = [torch.cuda.Event() for _ in self.segments]
        # each segment's input buffer (capacity B, the activation's own layout)
        self.x_in, self.rows_in, self.alive_in = [], [], []
        h = example
        with torch.no_grad():
            for a, e in self.segments:
                self.x_in.append(torch.zeros_like(h))
                self.rows_in.append(torch.full((b,), b, dtype=torch.int32, device=dev))
                self.alive_in.append(torch.zeros(b, dtype=torch.uint8, device=dev))
                for j in range(a, e + 1):
                    h = pipe.stages[j](h)
        self.x_in[0].copy_(example)  # run() without an input replays the example
        # segments whose last stage ends in a routed residual block compact in place
        self.fill = [k < len(self.segments) - 1 and b <= 8192 and can_run_into(pipe.stages[e])
                     and self.x_in[k + 1].is_contiguous(memory_format=torch.channels_last)
                     for k, (a, e) in enumerate(self.segments)]
        self.graphs = {}
        self.pool = torch.cuda.graph_pool_handle()
        self.out = BatchResult(self.slots.label[:b], self.slots.site[:b], self.slots.err[:b],
                               self.ramp_err[:, :b], self.ramp_label[:, :b], self.final_label[:b],
                               thresholds=self.th)

    def set_thresholds(self, thresholds):
        self.th.copy_(self.th.new_tensor([float(t) for t in thresholds]))

    def _segment(self, k: int, bb: int, host_count: bool = True):
        """Segment k at bucket bb: the eager body the graphs capture."""
        torch = nat.torch_cuda()
        a, e = self.segments[k]
        h = self.x_in[k][:bb]
        alive, rows = self.alive_in[k][:bb], self.rows_in[k][:bb]
        last = k == len(self.segments) - 1
        with torch.no_grad():
            for j in range(a, e):
                h = self.pipe.stages[j](h)
            if last:
                logits = self.pipe.stages[e](h).float()
                self.final_label.index_copy_(0, rows.long(), torch.argmax(logits, dim=1).to(torch.int32))
                exit_from_logits(logits.contiguous(), 2.0, conf="maxprob", site=self.R, alive=alive,
                                 slot=rows, slots=self.slots, compact=False)
                return
            if self.fill[k]:
                # the segment's last block writes straight into the next segment's
                # input buffer, which is then compacted in place: only survivors
                # above the live count move (a few rows), not every survivor
                h = run_into(self.pipe.stages[e], h, self.x_in[k + 1][:bb])
            else:
                h = self.pipe.stages[e](h)
            res = self.pipe.ramps[e](h, self.th[k:k + 1], alive=alive, slot=rows, slots=self.slots)
            scatter_signals(res.err, res.label, rows, self.ramp_err[k], self.ramp_label[k])
            if self.fill[k]:
                compact_fill(self.x_in[k + 1], res.keep, res.n_keep, bb, rows, self.B, self.rows_in[k + 1],
                             self.alive_in[k + 1], self.n_live[k:k + 1])
            else:
                compact_rows(h, res.keep, res.n_keep, out=self.x_in[k + 1])
                compact_meta(res.keep, res.n_keep, rows, self.B, self.B, self.rows_in[k + 1],
                             self.alive_in[k + 1], self.n_live[k:k + 1])
            if host_count:
                self.n_host[k:k + 1].copy_(self.n_live[k:k + 1], non_blocking=True)

    def _graph(self, k: int, bb: int):
        g = self.graphs.get((k, bb))
        if g is None:
            torch = nat.torch_cuda()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._segment(k, bb)  # warm-up (idempotent on the live state)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self.pool):
                self._segment(k, bb)
            self.graphs[(k, bb)] = g
        return g

    def device_chain(self):
        """Schedule the whole batch on the device (ee_seg_chain): every (segment,
        bucket) graph is captured once, and one executable graph runs segment 0
        at the full batch, then before each later segment a one-thread kernel
        reads the live count the previous segment left and a SWITCH node runs
        that segment at the smallest bucket >= it. No host round trip and no
        lag: each segment runs at the bucket of its own live rows."""
        if getattr(self, "_chain", None) is not None:
            return self._chain
        import ctypes

        torch = nat.torch_cuda()
        lib = nat.load_library()
        keep, ptrs = [], []

        def capture(body):
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                body()  # warm-up (idempotent on the live state)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g, pool=self.pool):
                body()
            keep.append(g)
            return g.raw_cuda_graph()

        reset = capture(self._reset)
        nb = len(self.buckets)
        for k in range(len(self.segments)):
            for bb in self.buckets:
                if k == 0 and bb != self.B:
                    ptrs.append(None)
                    continue
                ptrs.append(capture(lambda k=k, bb=bb: self._segment(k, bb, host_count=False)))
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        bk = (ctypes.c_int32 * nb)(*self.buckets)
        chain = ctypes.c_void_p()
        nat.check(lib.ee_seg_chain_create(arr, len(self.segments), nb, bk, self.n_live.data_ptr(), reset,
                                          ctypes.byref(chain)))
        self._chain_graphs = keep  # their memory pool backs the chain
        self._chain = chain
        return chain

    def run_device(self, x=None) -> BatchResult:
        """One compacted batch through device_chain(): a single graph launch."""
        torch = nat.torch_cuda()
        chain = self.device_chain()
        if x is not None:
            self.x_in[0].copy_(x)
        nat.check(nat.load_library().ee_seg_chain_launch(chain, nat.stream_handle(torch)))
        return self.out

    def __del__(self):
        chain = getattr(self, "_chain", None)
        if chain is not None:
            try:
                nat.load_library().ee_seg_chain_destroy(chain)
            except Exception:
                pass

    def bucket(self, n: int) -> int:
        for bb in self.buckets:
            if bb >= n:
                return bb
        return self.B

    def _reset(self):
        torch = nat.torch_cuda()
        self.n_live.zero_()  # a skipped segment reads as no live rows (device_chain)
        self.slots.label.fill_(-1)
        self.slots.site.fill_(-1)
        self.slots.err.fill_(float("nan"))
        self.ramp_err.fill_(float("nan"))
        self.ramp_label.fill_(-1)
        self.final_label.fill_(-1)
        self.alive_in[0].fill_(1)
        torch.arange(self.B, dtype=torch.int32, device="cuda", out=self.rows_in[0])

    def run(self, x=None) -> BatchResult:
        torch = nat.torch_cuda()
        if x is not None:
            self.x_in[0].copy_(x)
        if self.graphs.get("reset") is None:  # the table resets as one graph too
            self._reset()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self.pool):
                self._reset()
            self.graphs["reset"] = g
        self.graphs["reset"].replay()
        bb = self.B
        for k in range(len(self.segments)):
            if k >= 2:  # the count after segment k - 2 bounds segment k's live rows
                self.done[k - 2].synchronize()
                n = int(self.n_host[k - 2])
                if n == 0:
                    break
                bb = self.bucket(n)
            self._graph(k, bb).replay()
            self.done[k].record()
        return self.out


# ---------------------------------------------------------------- model builders
def fold_batchnorm(model):
    """Fold every eval-mode BatchNorm2d of a torchvision ResNet into the conv
    before it (w' = w * g / sqrt(v + eps) per output channel, b' = beta - mu * g /
    sqrt(v + eps)) and turn the BatchNorm into an identity, in place. The
    pipeline stages hold the same module objects, so they see the folded
    convolutions: one conv (+ bias) kernel instead of conv + BN kernels.
    (Model preparation only: it runs wherever the weights live.)"""
    import torch

    def fold(conv, bn):
        with torch.no_grad():
            scale = bn.weight.float() / torch.sqrt(bn.running_var.float() + bn.eps)
            conv.weight.mul_(scale.view(-1, 1, 1, 1).to(conv.weight.dtype))
            bias = bn.bias.float() - bn.running_mean.float() * scale
            if conv.bias is None:
                conv.bias = torch.nn.Parameter(bias.to(conv.weight.dtype))
            else:
                conv.bias.copy_(conv.bias.float() * scale + bias)
        bn.forward = lambda x: x  # the instance now passes activations through

    model.eval()
    fold(model.conv1, model.bn1)
    for layer in (model.layer1, model.layer2, model.layer3, model.layer4):
        for blk in layer:
            for i in (1, 2, 3):
                conv, bn = getattr(blk, f"conv{i}", None), getattr(blk, f"bn{i}", None)
                if conv is not None and bn is not None:
                    fold(conv, bn)
            if blk.downsample is not None:
                fold(blk.downsample[0], blk.downsample[1])
    return model


def prepare_bf16(model, channels_last: bool, route: bool = True):
    """The serving form of a backbone: bf16 weights and activations; CNNs
    additionally channels_last with BatchNorm folded into the convolutions.
    route: a ResNet's blocks then run on the repo's kernels (convnet.py:
    1x1 convolutions as tcgen05 GEMMs with bias / ReLU / shortcut fused, one
    fused epilogue pass after each spatial convolution); False keeps the
    library path (cuDNN convolutions + PyTorch elementwise kernels). In place."""
    import torch

    if channels_last:
        fold_batchnorm(model)
        model.to(memory_format=torch.channels_last)
    model.to(torch.bfloat16)
    if channels_last and route and hasattr(model, "layer4"):
        from paper_2312_05385_b200.convnet import route_resnet

        route_resnet(model)
    return model


def _calibrate_bn(model, shape, batches: int = 4, seed: int = 0):
    """Seeded train-mode passes so random-init BatchNorm statistics are sane."""
    torch = nat.torch_cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    model.train()
    with torch.no_grad():
        for _ in range(batches):
            model(torch.randn(*shape, generator=g, device="cuda"))
    model.eval()


def resnet18_cifar(num_classes: int = 10, ramp_sites=(0, 2, 3, 5, 6, 8), seed: int = 0,
                   conf: str = "maxprob"):
    """BASELINE config 1: ResNet-18, CIFAR shape (3x32x32), 6 ramps.

    Sites: 0 stem, 1 layer1.0, 2 layer1.1, 3 layer2.0, 4 layer2.1, 5 layer3.0,
    6 layer3.1, 7 layer4.0, 8 layer4.1 (SURVEY §8d picks stem, layer1.1,
    layer2.0, layer3.0, layer3.1, layer4.1)."""
    torch = nat.torch_cuda()
    import torchvision

    torch.manual_seed(seed)
    m = torchvision.models.resnet18(num_classes=num_classes)
    m.conv1 = torch.nn.Conv2d(3, 64, 3, 1, 1, bias=False)
    m.maxpool = torch.nn.Identity()
    m = m.cuda()
    _calibrate_bn(m, (64, 3, 32, 32), seed=seed)
    stem = torch.nn.Sequential(m.conv1, m.bn1, m.relu)
    blocks = [stem, m.layer1[0], m.layer1[1], m.layer2[0], m.layer2[1], m.layer3[0], m.layer3[1],
              m.layer4[0], m.layer4[1]]
    chans = [64, 64, 64, 128, 128, 256, 256, 512, 512]
    final = torch.nn.Sequential(m.avgpool, torch.nn.Flatten(), m.fc)
    g = torch.Generator().manual_seed(seed + 1)
    ramps = {}
    for s in ramp_sites:
        w = torch.randn(num_classes, chans[s], generator=g) / chans[s] ** 0.5
        ramps[s] = ExitController(w.cuda(), torch.zeros(num_classes).cuda(), conf=conf, site=len(ramps))
    names = ["stem", "layer1.0", "layer1.1", "layer2.0", "layer2.1", "layer3.0", "layer3.1",
             "layer4.0", "layer4.1"]
    return EEPipeline(blocks + [final], ramps, [names[s] for s in sorted(ramps)]), m


def resnet50_imagenet(seed: int = 0, conf: str = "maxprob", dtype=None, head_scale: float = 16.0):
    """BASELINE config 3: ResNet-50, 224x224, a ramp after each of the 16
    bottlenecks, 1000-class heads on the tensor-core GEMM path.

    Ramp FC init: N(0, (head_scale / sqrt(C))^2). Random-init pooled features
    barely vary across inputs, so at the usual 1/sqrt(C) every 1000-class
    confidence sits within ~1e-4 of 0.998 and every row of a batch is a 1e-5
    near-tie; at 16/sqrt(C) the per-ramp err spreads over ~0.05-0.1."""
    torch = nat.torch_cuda()
    import torchvision

    torch.manual_seed(seed)
    m = torchvision.models.resnet50().cuda()
    _calibrate_bn(m, (32, 3, 224, 224), seed=seed)
    stem = torch.nn.Sequential(m.conv1, m.bn1, m.relu, m.maxpool)
    blocks = []
    chans = []
    for layer, c in ((m.layer1, 256), (m.layer2, 512), (m.layer3, 1024), (m.layer4, 2048)):
        for blk in layer:
            blocks.append(blk)
            chans.append(c)
    stages = [torch.nn.Sequential(stem, blocks[0])] + blocks[1:]
    final = torch.nn.Sequential(m.avgpool, torch.nn.Flatten(), m.fc)
    g = torch.Generator().manual_seed(seed + 1)
    ramps = {}
    for s, c in enumerate(chans):
        w = torch.randn(1000, c, generator=g) * (head_scale / c ** 0.5)
        ramps[s] = LargeRampHead(w.cuda(), None, conf=conf, site=s)
    names = [f"bottleneck{s}" for s in range(len(chans))]
    return EEPipeline(stages + [final], ramps, names), m


def bert_base(seq: int = 128, seed: int = 0, conf: str = "entropy"):
    """BASELINE config 2: BERT-base-shape encoder (random init), a ramp after
    every layer on the token-0 hidden state (768 -> 2), entropy confidence."""
    torch = nat.torch_cuda()
    from transformers import BertConfig, BertModel

    torch.manual_seed(seed)
    cfg = BertConfig(attn_implementation="sdpa")
    bert = BertModel(cfg, add_pooling_layer=False).cuda().eval()

    class First:
        """Embeddings + encoder layer 0 (the first ramp sits after layer 0)."""

        def __init__(self, layer):
            self.layer = layer

        def __call__(self, ids):
            return self.layer(bert.embeddings(input_ids=ids))

    g = torch.Generator().manual_seed(seed + 1)
    layers = [BertLayerTC(l) for l in bert.encoder.layer]
    stages = [First(layers[0])] + layers[1:]
    heads = {}
    for s in range(len(layers)):
        w = torch.randn(2, cfg.hidden_size, generator=g) / cfg.hidden_size ** 0.5
        heads[s] = _Token0Head(ExitController(w.cuda(), torch.zeros(2).cuda(), conf=conf, site=s))
    final_w = (torch.randn(2, cfg.hidden_size, generator=g) / cfg.hidden_size ** 0.5).cuda()

    class Final(torch.nn.Module):
        """Final classifier on the token-0 hidden state (fp32 weight [2, 768])."""

        def __init__(self):
            super().__init__()
            self.weight = final_w

        def forward(self, h):
            return h[:, 0].float() @ self.weight.t()

    return EEPipeline(stages + [Final()], heads, [f"layer{s}" for s in range(len(layers))]), bert


class BertLayerTC:
    """One post-LN BERT encoder layer (the weights of a transformers BertLayer)
    with its four contractions on the repo's tcgen05 GEMMs (csrc/gemm.cu, A14):

        qkv = h Wqkv^T + b          one GEMM over the fused [3d, d] weight
        a   = SDPA(q, k, v)         (flash attention; not a GEMM this repo owns)
        x   = LN(h + a Wo^T + bo)   GEMM, then ee_add_layernorm_bf16 (add + LN, one pass)
        y   = LN(x + GELU(x W1^T + b1) W2^T + b2)   GELU fused into the W1 epilogue

    On bf16 weights (the serving form, ee_infer.prepare_bf16) every projection is
    a tcgen05 kernel; an fp32 model (the parity tests' reference configuration)
    runs the same math through torch. The fused weight copies are built on the
    first call after the dtype changes (before any CUDA-graph capture: the graph
    runner warms up first)."""

    def __init__(self, layer):
        self.layer = layer
        self._dtype = None

    def _prep(self):
        import torch

        L = self.layer
        sa, ao = L.attention.self, L.attention.output
        dt = sa.query.weight.dtype
        if dt == self._dtype:
            return
        self.n_head = sa.num_attention_heads
        self.wqkv = torch.cat([sa.query.weight, sa.key.weight, sa.value.weight]).contiguous()
        self.bqkv = torch.cat([sa.query.bias, sa.key.bias, sa.value.bias]).float().contiguous()
        self.wo, self.bo = ao.dense.weight.contiguous(), ao.dense.bias.float().contiguous()
        self.w1, self.b1 = L.intermediate.dense.weight.contiguous(), L.intermediate.dense.bias.float().contiguous()
        self.w2, self.b2 = L.output.dense.weight.contiguous(), L.output.dense.bias.float().contiguous()
        self.ln1, self.ln2 = ao.LayerNorm, L.output.LayerNorm
        self._dtype = dt

    def _add_ln(self, y, h, ln):
        """LN(h + y) (y is scratch and receives h + y)."""
        import torch

        if y.dtype != torch.bfloat16:
            return torch.nn.functional.layer_norm(h + y, ln.normalized_shape, ln.weight, ln.bias, ln.eps)
        out = torch.empty_like(y)
        d = y.shape[-1]
        nat.check(nat.load_library().ee_add_layernorm_bf16(
            y.data_ptr(), h.data_ptr(), ln.weight.data_ptr(), ln.bias.data_ptr(), float(ln.eps),
            y.numel() // d, d, out.data_ptr(), nat.stream_handle(torch)))
        return out

    def _linear(self, x, w, b, act=None):
        import torch
        import torch.nn.functional as F

        if x.dtype == torch.bfloat16:
            return gemm(x, w, b, act=act)
        y = F.linear(x, w, b)
        return F.gelu(y) if act == "gelu" else y

    def __call__(self, h):
        import torch
        import torch.nn.functional as F

        self._prep()
        h = h.contiguous()
        B, S, d = h.shape
        H = self.n_head
        qkv = self._linear(h, self.wqkv, self.bqkv).view(B, S, 3, H, d // H).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])
        a = a.transpose(1, 2).reshape(B, S, d)
        x = self._add_ln(self._linear(a, self.wo, self.bo), h, self.ln1)
        f = self._linear(x, self.w1, self.b1, act="gelu")
        return self._add_ln(self._linear(f, self.w2, self.b2), x, self.ln2)


class _Token0Head:
    """Ramp on a transformer layer: the head reads the token-0 hidden state."""

    def __init__(self, ctrl: ExitController):
        self.ctrl = ctrl

    def __call__(self, h, threshold, **kw):
        return self.ctrl(h[:, 0].contiguous(), threshold, **kw)

    @property
    def weight(self):
        return self.ctrl.weight

    @property
    def bias(self):
        return self.ctrl.bias

    @property
    def conf(self):
        return self.ctrl.conf
