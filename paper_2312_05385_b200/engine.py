"""Exit engine: exit decisions, accuracy and latency savings.

Public API of the reference's pkg/src/eesim/engine.py (EEConfig,
ExitOutcome, ServedRecord, WindowStats, decision_scores, WindowEvaluator,
evaluate_record, evaluate_window, optimal_exit), with the window evaluator
rebuilt around device-resident data:

  reference (engine.py:135-186)            here
  ---------------------------------------  ---------------------------------------
  packs records into numpy on every         packs once (trace.window_arrays) and
  construction, calls the Cython kernel     uploads scores (f64 [n, r]) and one
  with host arrays on every evaluation      u32 correctness bit row per sample to
                                            HBM; each evaluation ships only the
                                            (C, R) threshold rows
  decision_scores in numpy (k > 1)          K3 kernel on device (bit-identical)
  eval_thresholds / exit_sites (Cython)     K2 / K1 kernels via libeeb200.so

Exit rule (engine.py:189-220): a record exits at the first active ramp whose
decision score is strictly below the ramp's threshold; serve time is the
prefix through the exit layer plus every active ramp paid so far, or the full
model plus all ramps when nothing fires.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError, ValidationError
from paper_2312_05385_b200.graph import ModelProfile, RampSite
from paper_2312_05385_b200.trace import RequestRecord, WindowArrays, window_arrays


@dataclass(frozen=True)
class EEConfig:
    """Active ramps with thresholds, strictly increasing in topological order."""

    active: tuple[tuple[RampSite, float], ...]

    def __post_init__(self):
        last = -1
        for site, threshold in self.active:
            if site.topo_index <= last:
                raise ValidationError("active ramps must be strictly increasing in topological order")
            last = site.topo_index
            if not 0.0 <= threshold <= 1.0:
                raise ValidationError(f"threshold {threshold} outside [0, 1]")

    @property
    def sites(self) -> tuple[RampSite, ...]:
        return tuple(s for s, _ in self.active)

    @property
    def thresholds(self) -> tuple[float, ...]:
        return tuple(t for _, t in self.active)

    @property
    def positions(self) -> tuple[str, ...]:
        return tuple(s.position for s, _ in self.active)

    def threshold_at(self, position: str) -> float:
        for site, t in self.active:
            if site.position == position:
                return t
        raise KeyError(position)

    def with_thresholds(self, thresholds: Sequence[float] | Mapping[str, float]) -> "EEConfig":
        if isinstance(thresholds, Mapping):
            values = [float(thresholds[s.position]) for s, _ in self.active]
        else:
            if len(thresholds) != len(self.active):
                raise ParameterError("threshold count does not match active ramps")
            values = [float(t) for t in thresholds]
        return EEConfig(tuple((s, t) for (s, _), t in zip(self.active, values)))

    def ramp_overhead(self, batch: int = 1) -> float:
        return sum(s.ramp_ms(batch) for s, _ in self.active)

    def to_dict(self) -> dict:
        return {"ramps": [{"site": s.position, "threshold": t} for s, t in self.active]}


@dataclass(frozen=True)
class ExitOutcome:
    exit_site: str | None
    released_label: int
    correct: bool
    serve_ms: float


@dataclass(frozen=True)
class ServedRecord:
    """One request as served: trace record, outcome and batch size."""

    record: RequestRecord
    outcome: ExitOutcome
    batch: int = 1


@dataclass(frozen=True)
class WindowStats:
    accuracy: float
    mean_savings_ms: float
    exit_rates: Mapping[str, float]


def decision_scores(errs: np.ndarray, k: int = 1) -> np.ndarray:
    """Host twin of kernel K3: trailing mean of the last k active-ramp scores.

    k <= 1 (or a single ramp) returns `errs` itself, as engine.py:112-113 does."""
    if k <= 1 or errs.shape[1] <= 1:
        return errs
    r = errs.shape[1]
    csum = np.cumsum(errs, axis=1)
    out = np.empty_like(errs)
    for j in range(r):
        lo = max(0, j - k + 1)
        before = csum[:, lo - 1] if lo > 0 else 0.0
        out[:, j] = (csum[:, j] - before) / (j - lo + 1)
    return out


def serve_table(sites: Sequence[RampSite], profile: ModelProfile, batch: int) -> np.ndarray:
    """Serve time for releasing at ramp j (entry r: no exit), engine.py:124-132."""
    r = len(sites)
    serve = np.empty(r + 1)
    paid = 0.0
    for j, site in enumerate(sites):
        paid += site.ramp_ms(batch)
        serve[j] = site.prefix_ms(batch) + paid
    serve[r] = profile.model_latency(batch) + paid if r else profile.model_latency(batch)
    return serve


def _pack_bits(correct: np.ndarray) -> np.ndarray:
    """u8 [n, r+1] (0/1) -> u32 [n] with bit j = column j."""
    n, r1 = correct.shape
    padded = np.zeros((n, 32), dtype=np.uint8)
    padded[:, :r1] = correct != 0
    return np.packbits(padded, axis=1, bitorder="little").view("<u4").reshape(n)


# Sweeps over an evaluator's own (immutable) device window are launched with
# EE_MODE_FLAG_RESIDENT; False forces plain stream-ordered launches (A/B).
RESIDENT_OVERLAP = True

class WindowEvaluator:
    """Device-resident window: upload once, score many threshold configs.

    Attributes mirror the reference (`records`, `sites`, `profile`, `batch`,
    `serve`, `vanilla_ms`, host views `scores` / `correct_ext`); the device
    tensors are `d_scores` (f64 [n, r]) and `d_bits` (u32 [n]).
    `mode` selects the evaluation kernel: "exact" (bit-identical to the
    Cython loop), "hist" (integer histograms) or "auto" (exact up to 4096
    samples).
    """

    def __init__(self, records: Sequence[RequestRecord], sites: Sequence[RampSite],
                 profile: ModelProfile, batch: int = 1, k: int = 1, *, mode: str | None = None):
        if not records:
            raise ParameterError("window is empty")
        self.records = tuple(records)
        self._setup(window_arrays(self.records, sites), sites, profile, batch, k, mode)

    @classmethod
    def from_arrays(cls, arrays: WindowArrays, sites: Sequence[RampSite], profile: ModelProfile,
                    batch: int = 1, k: int = 1, *, mode: str | None = None,
                    records: Sequence[RequestRecord] | None = None) -> "WindowEvaluator":
        """Build from columnar arrays (no per-record Python work)."""
        if arrays.n == 0:
            raise ParameterError("window is empty")
        if arrays.r != len(sites):
            raise ParameterError(f"arrays have {arrays.r} ramps, {len(sites)} sites given")
        ev = cls.__new__(cls)
        ev.records = tuple(records) if records is not None else None
        ev._setup(arrays, sites, profile, batch, k, mode)
        return ev

    def _setup(self, arrays: WindowArrays, sites, profile, batch, k, mode):
        from paper_2312_05385_b200 import kernels

        self.sites = tuple(sites)
        self.profile = profile
        self.batch = batch
        self.k = k
        self.n = arrays.n
        self.r = len(self.sites)
        if self.r > nat.MAX_RAMPS:
            raise ParameterError(f"{self.r} ramps exceed the supported maximum of {nat.MAX_RAMPS}")
        self.mode = mode
        self._mode_code = kernels._mode_code(mode)
        self.serve = serve_table(self.sites, profile, batch)
        self.vanilla_ms = profile.model_latency(batch)
        self._arrays = arrays
        torch = nat.torch_cuda()
        self._torch = torch
        lib = nat.load_library()
        errs = np.ascontiguousarray(arrays.errs, dtype=np.float64)
        d_errs = torch.from_numpy(errs).to("cuda")
        if k > 1 and self.r > 1:
            d_scores = torch.empty_like(d_errs)
            nat.check(lib.ee_decision_scores(d_errs.data_ptr(), self.n, self.r, k,
                                             d_scores.data_ptr(), nat.stream_handle(torch)))
            self.d_scores = d_scores
        else:
            self.d_scores = d_errs
        bits = _pack_bits(arrays.correct)
        self.d_bits = torch.from_numpy(bits.view(np.int32)).to("cuda")
        self._scores_host = None
        # The window is immutable from here on: once its producers have finished,
        # sweeps may overlap the previous sweep on the stream (EE_MODE_FLAG_RESIDENT).
        torch.cuda.current_stream().synchronize()

    # host views kept for API parity with the reference attributes
    @property
    def scores(self) -> np.ndarray:
        if self._scores_host is None:
            self._scores_host = self.d_scores.cpu().numpy()
        return self._scores_host

    @property
    def correct_ext(self) -> np.ndarray:
        return self._arrays.correct_ext()

    def _eval_device(self, th: np.ndarray, want_hist: bool = False, mode_code: int | None = None,
                     counts_only: bool = False):
        torch = self._torch
        lib = nat.load_library()
        c = th.shape[0]
        if counts_only:
            # hist then ok in ONE int64 buffer: a cross-rank all-reduce sums it in place
            buf = torch.empty(c * (self.r + 2), dtype=torch.int64, device="cuda")
            acc = sav = None
            hist = buf[: c * (self.r + 1)].view(c, self.r + 1)
            ok = buf[c * (self.r + 1):]
        else:
            out = torch.empty((3, c), dtype=torch.float64, device="cuda")  # one allocation per call
            acc, sav = out[0], out[1]
            ok = out[2].view(torch.int64)
            hist = torch.empty((c, self.r + 1), dtype=torch.int64, device="cuda") if want_hist else None
        nat.check(lib.ee_eval_thresholds(
            nat.workspace(), nat.ptr(self.d_scores), self.d_bits.data_ptr(), self.n, self.r,
            self.serve.ctypes.data, float(self.vanilla_ms), th.ctypes.data if th.size else None,
            c, (self._mode_code if mode_code is None else mode_code)
            | (nat.MODE_FLAG_RESIDENT if RESIDENT_OVERLAP else 0),
            nat.ptr(hist), ok.data_ptr(),
            nat.ptr(acc), nat.ptr(sav), nat.stream_handle(torch)))
        return acc, sav, ok, hist

    def evaluate_many(self, thresholds: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """(accuracy, mean savings) for each row of a (C, R) threshold matrix."""
        th = np.ascontiguousarray(thresholds, dtype=np.float64)
        if th.ndim != 2 or th.shape[1] != self.r:
            raise ParameterError(f"thresholds must be (C, {self.r}), got {th.shape}")
        if th.shape[0] == 0:
            return np.empty(0), np.empty(0)
        acc, sav, _, _ = self._eval_device(th)
        return acc.cpu().numpy(), sav.cpu().numpy()

    def histograms(self, thresholds: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Exact integer exit-site histograms (C, R+1) and correct counts (C,)."""
        th = np.ascontiguousarray(thresholds, dtype=np.float64)
        if th.ndim != 2 or th.shape[1] != self.r:
            raise ParameterError(f"thresholds must be (C, {self.r}), got {th.shape}")
        _, _, ok, hist = self._eval_device(th, want_hist=True, mode_code=nat.MODE_HIST)
        return hist.cpu().numpy(), ok.cpu().numpy()

    def evaluate_lattice(self, vals: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """acc/sav for every point of vals^r in lexicographic order, never materialised."""
        torch = self._torch
        lib = nat.load_library()
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        c = len(vals) ** self.r
        acc = torch.empty(c, dtype=torch.float64, device="cuda")
        sav = torch.empty(c, dtype=torch.float64, device="cuda")
        nat.check(lib.ee_eval_lattice(
            nat.workspace(), nat.ptr(self.d_scores), self.d_bits.data_ptr(), self.n, self.r,
            self.serve.ctypes.data, float(self.vanilla_ms), vals.ctypes.data, len(vals),
            acc.data_ptr(), sav.data_ptr(), nat.stream_handle(torch)))
        return acc.cpu().numpy(), sav.cpu().numpy()

    def exit_indices(self, thresholds: Sequence[float]) -> np.ndarray:
        """Per-record exit index (len(sites) = no exit) for one config."""
        if self.r == 0:
            return np.zeros(self.n, dtype=np.int64)
        torch = self._torch
        th = torch.as_tensor(np.ascontiguousarray(thresholds, dtype=np.float64)).to("cuda")
        if th.numel() != self.r:
            raise ParameterError(f"expected {self.r} thresholds, got {th.numel()}")
        out = torch.empty(self.n, dtype=torch.int64, device="cuda")
        nat.check(nat.load_library().ee_exit_sites(
            nat.ptr(self.d_scores), self.n, self.r, th.data_ptr(), out.data_ptr(),
            nat.stream_handle(torch)))
        return out.cpu().numpy()

    def evaluate(self, thresholds: Sequence[float]) -> WindowStats:
        r = self.r
        th = np.asarray(thresholds, dtype=np.float64).reshape(1, r)
        acc, sav = self.evaluate_many(th)
        idx = self.exit_indices(thresholds)
        counts = np.bincount(idx, minlength=r + 1)
        rates = {site.position: counts[j] / self.n for j, site in enumerate(self.sites)}
        return WindowStats(float(acc[0]), float(sav[0]), rates)


def evaluate_record(record: RequestRecord, config: EEConfig, profile: ModelProfile,
                    batch: int = 1, k: int = 1) -> ExitOutcome:
    """Exit decision and serve time for one record (engine.py:189-220)."""
    paid = 0.0
    recent: list[float] = []
    signals = record.ramp_signals
    for site, threshold in config.active:
        paid += site.ramp_ms(batch)
        err = signals[site.position].err
        recent.append(err)
        if len(recent) > k:
            del recent[0]
        score = err if k <= 1 else sum(recent) / len(recent)
        if score < threshold:
            label = signals[site.position].label
            return ExitOutcome(site.position, label, label == record.final_label,
                               site.prefix_ms(batch) + paid)
    return ExitOutcome(None, record.final_label, True, profile.model_latency(batch) + paid)


def evaluate_window(records: Sequence[RequestRecord], config: EEConfig, profile: ModelProfile,
                    *, batch: int = 1, k: int = 1) -> WindowStats:
    """Accuracy, mean savings vs vanilla and per-ramp exit rates over a window."""
    if not records:
        raise ParameterError("evaluate_window requires a nonempty window")
    ev = WindowEvaluator(records, config.sites, profile, batch=batch, k=k)
    return ev.evaluate(config.thresholds)


def optimal_exit(record: RequestRecord, sites: Sequence[RampSite]) -> str | None:
    """Earliest site whose label matches the final label (upper-bound baseline)."""
    for site in sites:
        if record.ramp_signals[site.position].label == record.final_label:
            return site.position
    return None
