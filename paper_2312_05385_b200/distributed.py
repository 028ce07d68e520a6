"""Sample-sharded threshold sweep across GPUs.

Samples are independent, so rank g owns rows [g*N/G, (g+1)*N/G) of the window
and computes integer exit-site histograms for every candidate on its shard
(HIST mode). The only exchange is one all-reduce (sum) of C*(R+2) int64
counters — histograms plus correct counts — over NCCL; every rank then
finalises identical acc/sav from the global counts, so results are
bit-identical for any world size. One process per GPU, torch.distributed for
the plumbing.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.graph import ModelProfile, RampSite
from paper_2312_05385_b200.trace import WindowArrays


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) sample range of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def reduce_counts(hist, ok, group=None):
    """Sum per-shard int64 histograms and correct counts across ranks (in place).

    One collective: the two tensors are packed into a single buffer so the
    exchange is a single all-reduce of C*(R+2) int64."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return hist, ok
    c, r1 = hist.shape
    base = hist.untyped_storage().data_ptr()
    if (hist.is_contiguous() and ok.is_contiguous() and hist.data_ptr() == base
            and ok.data_ptr() == base + hist.numel() * 8
            and hist.untyped_storage().nbytes() == (hist.numel() + ok.numel()) * 8):
        # already one buffer (WindowEvaluator counts-only): all-reduce it in place
        buf = torch.empty(0, dtype=torch.int64, device=hist.device).set_(
            hist.untyped_storage(), 0, (hist.numel() + ok.numel(),))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        return hist, ok
    buf = torch.cat([hist.reshape(-1), ok.reshape(-1)])
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf[: c * r1].view(c, r1), buf[c * r1:]


class ShardedSweep:
    """Per-rank device window over this rank's sample shard plus the reduction."""

    def __init__(self, arrays: WindowArrays, sites: Sequence[RampSite], profile: ModelProfile,
                 *, rank: int = 0, world: int = 1, n_total: int | None = None, group=None,
                 already_sharded: bool = False, overlap_comm: bool = False, comm_stream=None):
        """overlap_comm: the all-reduce and finalisation of each sweep run on a
        side stream, so a stream of sweeps overlaps sweep k+1 with the exchange
        of sweep k. Results are then ready once `self.ready` (an event) has
        completed; `join()` makes the current stream wait for all of them.
        Sweeps sharing a process group must share `comm_stream` (collectives
        on one communicator stay in one order)."""
        self.n_total = int(n_total if n_total is not None else arrays.n)
        if not already_sharded:
            lo, hi = shard_range(arrays.n, rank, world)
            arrays = WindowArrays(arrays.errs[lo:hi], arrays.correct[lo:hi])
        self.group = group
        self.local = WindowEvaluator.from_arrays(arrays, sites, profile, mode="hist")
        self.r = len(sites)
        self.overlap_comm = overlap_comm
        self.comm = comm_stream
        self.ready = None

    def counts(self, thresholds: np.ndarray):
        """Global (hist [C, R+1], ok [C]) as int64 device tensors."""
        th = np.ascontiguousarray(thresholds, dtype=np.float64)
        _, _, ok, hist = self.local._eval_device(th, want_hist=True, mode_code=nat.MODE_HIST,
                                                 counts_only=True)
        return reduce_counts(hist, ok, self.group)

    def _single(self) -> bool:
        import torch.distributed as dist

        return not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(self.group) == 1

    def evaluate_many(self, thresholds: np.ndarray, *, to_host: bool = True):
        torch = self.local._torch
        if self._single():  # nothing to exchange: one fused evaluation
            th = np.ascontiguousarray(thresholds, dtype=np.float64)
            acc, sav, _, _ = self.local._eval_device(th, mode_code=nat.MODE_HIST)
            return (acc.cpu().numpy(), sav.cpu().numpy()) if to_host else (acc, sav)
        if not self.overlap_comm:
            hist, ok = self.counts(thresholds)
            acc, sav = self._finalize(torch, hist, ok)
        else:
            th = np.ascontiguousarray(thresholds, dtype=np.float64)
            _, _, ok, hist = self.local._eval_device(th, want_hist=True, mode_code=nat.MODE_HIST,
                                                     counts_only=True)
            if self.comm is None:
                self.comm = torch.cuda.Stream()
            swept = torch.cuda.Event()
            swept.record()
            with torch.cuda.stream(self.comm):
                self.comm.wait_event(swept)
                hist, ok = reduce_counts(hist, ok, self.group)
                acc, sav = self._finalize(torch, hist, ok)
            for t in (hist, ok, acc, sav):  # in use on the side stream: no early reuse
                t.record_stream(self.comm)
            self.ready = torch.cuda.Event()
            self.ready.record(self.comm)
            if to_host:
                self.ready.synchronize()
        if to_host:
            return acc.cpu().numpy(), sav.cpu().numpy()
        return acc, sav

    def join(self) -> None:
        """Make the current stream wait for every overlapped exchange issued so far."""
        import torch

        if self.comm is not None:
            torch.cuda.current_stream().wait_stream(self.comm)

    def _finalize(self, torch, hist, ok):
        c = hist.shape[0]
        acc = torch.empty(c, dtype=torch.float64, device="cuda")
        sav = torch.empty(c, dtype=torch.float64, device="cuda")
        ev = self.local
        nat.check(nat.load_library().ee_finalize_hist(
            nat.workspace(), hist.data_ptr(), ok.data_ptr(), c, self.r, self.n_total,
            ev.serve.ctypes.data, float(ev.vanilla_ms), acc.data_ptr(), sav.data_ptr(),
            nat.stream_handle(torch)))
        return acc, sav


WINDOW_ACC_WORDS = 2178  # EE_WINDOW_ACC_WORDS (include/eeb200.h)


class WindowStream:
    """A stream of config-4 sweeps over resident, sample-sharded windows as ONE
    persistent counting launch per call (k_diag3_windows_db: tables built once,
    each window's fold overlapped with the next window's stream), ONE
    all-reduce of the K per-window totals (K x 2178 int64) when the group has
    more than one rank, and one finalisation with the global sample count
    (ee_windows_counts / ee_windows_finalize). Every buffer is allocated here,
    so a call can be captured in a CUDA graph. Diagonal candidate rows only
    (<= 64 distinct thresholds, even r <= 16). Results equal evaluating each
    full window on its own, bit for bit."""

    def __init__(self, sweeps: Sequence["ShardedSweep"], order=None, *, group=None):
        import torch

        if not sweeps:
            raise ParameterError("no windows")
        s0 = sweeps[0].local
        for sw in sweeps[1:]:
            e = sw.local
            if e.n != s0.n or e.r != s0.r or not np.array_equal(e.serve, s0.serve) or \
                    e.vanilla_ms != s0.vanilla_ms or sw.n_total != sweeps[0].n_total:
                raise ParameterError("windows must share n, r, serve table and vanilla latency")
        order = list(range(len(sweeps))) if order is None else [int(i) for i in order]
        if not order or any(i < 0 or i >= len(sweeps) for i in order):
            raise ParameterError("bad window order")
        self.sweeps, self.order, self.group = list(sweeps), order, group
        self.n, self.r, self.n_total = s0.n, s0.r, sweeps[0].n_total
        self.serve, self.vanilla = s0.serve, float(s0.vanilla_ms)
        self.sl = torch.tensor([nat.ptr(sweeps[i].local.d_scores) for i in order], dtype=torch.int64,
                               device="cuda")
        self.bl = torch.tensor([sweeps[i].local.d_bits.data_ptr() for i in order], dtype=torch.int64,
                               device="cuda")
        self.accw = torch.zeros((len(order), WINDOW_ACC_WORDS), dtype=torch.int64, device="cuda")
        self.acc = self.sav = None

    def run(self, thresholds):
        """acc, sav [K, C] (CUDA f64) for the candidate rows `thresholds` (C, r)."""
        import torch
        import torch.distributed as dist

        th = np.ascontiguousarray(thresholds, dtype=np.float64)
        if th.ndim != 2 or th.shape[1] != self.r:
            raise ParameterError(f"thresholds must be (C, {self.r})")
        c, k = th.shape[0], len(self.order)
        if self.acc is None or self.acc.shape != (k, c):
            self.acc = torch.empty((k, c), dtype=torch.float64, device="cuda")
            self.sav = torch.empty((k, c), dtype=torch.float64, device="cuda")
        lib, st = nat.load_library(), nat.stream_handle(torch)
        nat.check(lib.ee_windows_counts(nat.workspace(), self.sl.data_ptr(), self.bl.data_ptr(), k,
                                        self.n, self.r, th.ctypes.data, c, self.accw.data_ptr(), st))
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(self.accw, op=dist.ReduceOp.SUM, group=self.group)
        nat.check(lib.ee_windows_finalize(nat.workspace(), self.accw.data_ptr(), k, self.n_total, self.r,
                                          self.serve.ctypes.data, self.vanilla, th.ctypes.data, c,
                                          self.acc.data_ptr(), self.sav.data_ptr(), st))
        return self.acc, self.sav


def evaluate_windows(sweeps: Sequence["ShardedSweep"], thresholds: np.ndarray, *, group=None,
                     to_host: bool = True):
    """acc, sav [K, C] for K windows sharded the same way (one ShardedSweep per
    window on this rank): K counts-only sweeps into one packed int64 buffer,
    ONE all-reduce of K * C * (R + 2) counters for all of them, then K
    finalisations — the exchange's latency is paid once per K windows instead
    of once per window. Bit-identical to K separate evaluate_many calls."""
    import torch
    import torch.distributed as dist

    if not sweeps:
        raise ParameterError("no windows")
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    r = sweeps[0].r
    if th.ndim != 2 or th.shape[1] != r or any(sw.r != r for sw in sweeps):
        raise ParameterError("every window must have the thresholds' ramp count")
    c = th.shape[0]
    parts = []
    for sw in sweeps:
        _, _, ok, hist = sw.local._eval_device(th, want_hist=True, mode_code=nat.MODE_HIST,
                                               counts_only=True)
        parts += [hist.reshape(-1), ok.reshape(-1)]
    flat = torch.cat(parts)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    per = c * (r + 2)
    accs, savs = [], []
    for k, sw in enumerate(sweeps):
        blk = flat[k * per:(k + 1) * per]
        a, v = sw._finalize(torch, blk[: c * (r + 1)].view(c, r + 1), blk[c * (r + 1):])
        accs.append(a)
        savs.append(v)
    acc, sav = torch.stack(accs), torch.stack(savs)
    return (acc.cpu().numpy(), sav.cpu().numpy()) if to_host else (acc, sav)


def eval_thresholds_host_sharded(scores, correct_ext, serve, vanilla, thresholds, *, n_total: int,
                                 group=None):
    """Drop-in `eval_thresholds` over this rank's host-resident sample shard:
    H2D of the shard, per-shard histograms, one all-reduce, identical
    finalisation on every rank; returns host (acc, sav) for all candidates."""
    from paper_2312_05385_b200 import kernels

    torch = nat.torch_cuda()
    lib = nat.load_library()
    scores = kernels._check_view(scores, 2, "scores")
    correct_ext = kernels._check_view(correct_ext, 2, "correct_ext")
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    serve = np.ascontiguousarray(serve, dtype=np.float64)
    n, r = scores.shape
    c = th.shape[0]
    if tuple(correct_ext.shape) != (n, r + 1) or serve.shape != (r + 1,) or th.ndim != 2 or th.shape[1] != r:
        raise ParameterError("shard shapes disagree: scores (n, r), correct_ext (n, r+1), serve (r+1,), th (c, r)")
    hist = torch.empty((c, r + 1), dtype=torch.int64, device="cuda")
    ok = torch.empty(c, dtype=torch.int64, device="cuda")
    acc = torch.empty(c, dtype=torch.float64, device="cuda")
    sav = torch.empty(c, dtype=torch.float64, device="cuda")
    st = nat.stream_handle(torch)
    # correct_ext packed to bit rows on the host cores while the scores stream
    # (8r + 4 bytes per sample over PCIe, as the 1-GPU host path); a non-binary
    # entry raises ValueError (EE_ERR_NOT_BINARY) before any exchange
    bad = None
    try:
        nat.check(lib.ee_eval_counts_host(
            nat.workspace(), scores.ctypes.data if scores.size else None,
            correct_ext.ctypes.data if correct_ext.size else None, n, r,
            th.ctypes.data if th.size else None, c, hist.data_ptr(), ok.data_ptr(), 0, st))
    except ValueError as e:  # still take part in the exchange: the other ranks wait on it
        bad = e
        hist.zero_()
        ok.zero_()
    hist, ok = reduce_counts(hist, ok, group)
    nat.check(lib.ee_finalize_hist(nat.workspace(), hist.data_ptr(), ok.data_ptr(), c, r, n_total,
                                   serve.ctypes.data, float(vanilla), acc.data_ptr(),
                                   sav.data_ptr(), st))
    if bad is not None:
        raise bad
    return acc.cpu().numpy(), sav.cpu().numpy()
