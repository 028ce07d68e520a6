"""TEST INFRASTRUCTURE ONLY: a plain-Python restatement of the reference's
token-level early-exit timeline (pkg/src/eesim/generative.py), used as the
checker for the GPU decoder in paper_2312_05385_b200/generative.py. Nothing
on the product path imports this module.

Pinned against the reference itself in tests/test_generative_oracle.py
(imports the installed reference from baseline/_ref when present).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence


def exit_index(signals, config, k: int) -> int | None:
    """generative.py:157-167 (_exit_index): first active ramp whose (k-mean) err
    is strictly below its threshold."""
    window: list[float] = []
    for j, (site, threshold) in enumerate(config.active):
        err = signals[site.position].err
        window.append(err)
        if len(window) > k:
            window.pop(0)
        score = err if k <= 1 else sum(window) / len(window)
        if score < threshold:
            return j
    return None


@dataclass
class Stat:
    index: int
    tpt_ms: float
    exit_site: str | None
    correct: bool


@dataclass
class Flush:
    site: str
    tokens: int
    penalty: float
    duration_ms: float
    kind: str  # "cap" | "carry" | "end"


def sequence_timeline(tokens: Sequence, profile, config, *, flush_cap: int = 4,
                      penalty: Callable[[int], float] = lambda b: 1.0, k: int = 1):
    """_SequenceSim.run (generative.py:202-261) for one sequence under a fixed
    config: per-token (tpt, exit site, correct) and the flush events, plus the
    critical-path clock. `tokens[i]` needs `.ramp_signals` {position:
    RampSignal} and `.final_token`."""
    total = profile.model_latency(1)
    clock = 0.0
    stats: list[Stat] = []
    flushes: list[Flush] = []
    deferred: dict[str, int] = {}

    def suffix(position):
        return total - profile.prefix_latency(position, 1)

    def flush(position, kind):
        nonlocal clock
        count = deferred.pop(position, 0)
        if not count:
            return
        mult = penalty(count)
        per = mult * suffix(position)
        clock += per
        flushes.append(Flush(position, count, mult, per, kind))

    for i, tok in enumerate(tokens):
        j = exit_index(tok.ramp_signals, config, k)
        if j is not None:
            site = config.sites[j]
            ramp_cost = sum(s.ramp_ms(1) for s in config.sites[: j + 1])
            tpt = site.prefix_ms(1) + ramp_cost
            clock += tpt
            label = tok.ramp_signals[site.position].label
            stats.append(Stat(i, tpt, site.position, label == tok.final_token))
            deferred[site.position] = deferred.get(site.position, 0) + 1
            if deferred[site.position] >= flush_cap:
                flush(site.position, "cap")
            continue
        ramp_cost = config.ramp_overhead(1)
        if not deferred:
            tpt = total + ramp_cost
            stats.append(Stat(i, tpt, None, True))
            clock += tpt
            continue
        points = [(s.position, profile.prefix_latency(s.position, 1))
                  for s, _ in config.active if deferred.get(s.position)]
        tpt = points[0][1]
        batch = 1
        shares = {pos: 0.0 for pos, _ in points}
        for idx, (pos, prefix_ms) in enumerate(points):
            batch += deferred[pos]
            seg_end = points[idx + 1][1] if idx + 1 < len(points) else total
            seg = penalty(batch) * (seg_end - prefix_ms)
            tpt += seg
            for p, _ in points[: idx + 1]:
                shares[p] += seg
        tpt += ramp_cost
        stats.append(Stat(i, tpt, None, True))
        clock += tpt
        for pos, _ in points:
            count = deferred.pop(pos)
            flushes.append(Flush(pos, count, penalty(1 + count), shares[pos], "carry"))
    for site, _ in config.active:
        flush(site.position, "end")
    return stats, flushes, clock
