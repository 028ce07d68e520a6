"""Per-ramp utilities: exit-site histograms turned into
savings / overheads / exit rates.

API of the reference's pkg/src/eesim/ramps.py:34-141 (RampUtility,
UtilityReport, score_utilities, estimate_utilities). estimate_utilities takes
the per-record exit indices from the GPU (kernel K1 through the device
window) and then folds them on the host in record order, so every float sum
is accumulated exactly as the reference accumulates it. Ramp adjustment
(Algorithm 2, ramps.py:144-371) is control logic outside the GPU path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from paper_2312_05385_b200.engine import EEConfig, ServedRecord, WindowEvaluator
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.graph import ModelProfile
from paper_2312_05385_b200.trace import RequestRecord


@dataclass(frozen=True)
class RampUtility:
    site: str
    savings_ms: float
    overheads_ms: float
    exit_rate: float

    @property
    def utility_ms(self) -> float:
        return self.savings_ms - self.overheads_ms


@dataclass(frozen=True)
class UtilityReport:
    ramps: tuple[RampUtility, ...]
    period_len: int
    mean_savings_ms: float

    def utility_of(self, position: str) -> RampUtility:
        for u in self.ramps:
            if u.site == position:
                return u
        raise KeyError(position)

    def to_dict(self) -> dict:
        return {
            "period_len": self.period_len,
            "mean_savings_ms": self.mean_savings_ms,
            "ramps": [
                {"site": u.site, "savings_ms": u.savings_ms, "overheads_ms": u.overheads_ms,
                 "exit_rate": u.exit_rate, "utility_ms": u.utility_ms}
                for u in self.ramps
            ],
        }


def _fold(exit_idx: Sequence[int], saving_of, overhead_of, n_ramps: int, total_len: int, sites):
    savings = [0.0] * n_ramps
    overheads = [0.0] * n_ramps
    exits = [0] * n_ramps
    total = 0.0
    for row, i in enumerate(exit_idx):
        s = saving_of(row, i)
        total += s
        if i < n_ramps:
            savings[i] += s
            exits[i] += 1
        for j in range(n_ramps):
            if i > j:  # passed ramp j without exiting there
                overheads[j] += overhead_of(row, j)
    ramps = tuple(RampUtility(site.position, savings[j], overheads[j], exits[j] / total_len)
                  for j, site in enumerate(sites))
    return UtilityReport(ramps, total_len, total / total_len)


def score_utilities(period: Sequence[ServedRecord], config: EEConfig,
                    profile: ModelProfile) -> UtilityReport:
    """Per-ramp utility over served requests at their served batch sizes."""
    if not period:
        raise ParameterError("score_utilities requires a nonempty period")
    order = {site.position: j for j, site in enumerate(config.sites)}
    n = len(config.sites)
    idx = [order.get(sr.outcome.exit_site, n) if sr.outcome.exit_site else n for sr in period]

    def saving(row, _i):
        sr = period[row]
        return profile.model_latency(sr.batch) - sr.outcome.serve_ms

    def overhead(row, j):
        return config.sites[j].ramp_ms(period[row].batch)

    return _fold(idx, saving, overhead, n, len(period), config.sites)


def estimate_utilities(history: Sequence[RequestRecord], config: EEConfig, profile: ModelProfile,
                       k: int = 1, *, evaluator: WindowEvaluator | None = None) -> UtilityReport:
    """Offline utility estimate at batch 1; exit indices come from the GPU."""
    ev = evaluator or WindowEvaluator(history, config.sites, profile, batch=1, k=k)
    idx = ev.exit_indices(config.thresholds)
    n = len(config.sites)
    vanilla = ev.vanilla_ms
    serve = ev.serve
    ramp_ms = [s.ramp_ms(1) for s in config.sites]
    return _fold(idx.tolist(), lambda _row, i: vanilla - serve[i], lambda _row, j: ramp_ms[j], n,
                 ev.n, config.sites)
