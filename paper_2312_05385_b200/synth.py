"""Columnar window synthesis at 1M-record scale.

`synthesize_window` returns the same signals as trace.synthesize_workload
(the reference generator, pkg/src/eesim/trace.py:164-227) for the same seed,
but as a WindowArrays and through the native replay loop ee_synth_columns
(csrc/synth.cpp) over numpy's raw PCG64 stream: ~1 s per 1M x 12 instead of
~64 s of per-record Python (host-only; no GPU involved).
"""

from __future__ import annotations

import ctypes
from typing import Mapping, Sequence

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.graph import ModelProfile, RampSite, find_feasible_sites
from paper_2312_05385_b200.trace import WindowArrays, _synth_params

_CHUNK = 1 << 22  # raw draws per refill


def synthesize_columns(profile: ModelProfile, n: int, continuity: float,
                       agreement_curve: Mapping[str, float], seed: int, *,
                       miscalibration: float = 0.05,
                       late_agreement_curve: Mapping[str, float] | None = None,
                       late_miscalibration: float | None = None, n_labels: int = 10):
    """(sites, errs f64 [n, S], labels i32 [n, S], finals i32 [n]) over all feasible sites."""
    sites, early, late, miscal_late = _synth_params(
        profile, continuity, agreement_curve, miscalibration, late_agreement_curve,
        late_miscalibration, n_labels)
    lib = nat.load_library()
    s = len(sites)
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    bg = rng.bit_generator
    errs = np.empty((n, s))
    labels = np.empty((n, s), dtype=np.int32)
    finals = np.empty(n, dtype=np.int32)
    early_a = np.ascontiguousarray(early, dtype=np.float64)
    late_a = np.ascontiguousarray(late, dtype=np.float64)
    pos = ctypes.c_int64(0)
    has32 = ctypes.c_int32(0)
    buf = ctypes.c_uint32(0)
    d_prev = ctypes.c_double(0.0)
    t_end = ctypes.c_int64(0)
    t = 0
    raw = np.empty(0, dtype=np.uint64)
    while t < n:
        raw = np.concatenate([raw[pos.value:], bg.random_raw(_CHUNK)])
        pos.value = 0
        nat.check(lib.ee_synth_columns(
            raw.ctypes.data, raw.size, ctypes.byref(pos), ctypes.byref(has32), ctypes.byref(buf),
            u.ctypes.data, n, t, ctypes.byref(t_end), ctypes.byref(d_prev), s,
            early_a.ctypes.data, late_a.ctypes.data, int(late_agreement_curve is not None),
            float(continuity), float(miscalibration), float(miscal_late), int(n_labels),
            errs.ctypes.data, labels.ctypes.data, finals.ctypes.data))
        t = t_end.value
    return sites, errs, labels, finals


def to_window(sites_all: Sequence[RampSite], errs, labels, finals,
              sites: Sequence[RampSite] | None = None) -> WindowArrays:
    """Select ramp columns and build the correctness matrix (engine.py:154-159)."""
    if sites is None:
        cols = list(range(len(sites_all)))
    else:
        index = {x.position: j for j, x in enumerate(sites_all)}
        cols = [index[x.position] for x in sites]
    e = np.ascontiguousarray(errs[:, cols])
    n, r = e.shape
    correct = np.ones((n, r + 1), dtype=np.uint8)
    correct[:, :r] = labels[:, cols] == finals[:, None]
    return WindowArrays(e, correct)


def synthesize_window(profile: ModelProfile, n: int, continuity: float,
                      agreement_curve: Mapping[str, float], seed: int, *,
                      sites: Sequence[RampSite] | None = None, **kw) -> WindowArrays:
    sites_all, errs, labels, finals = synthesize_columns(profile, n, continuity, agreement_curve,
                                                         seed, **kw)
    return to_window(sites_all, errs, labels, finals, sites)


def config4_profile() -> ModelProfile:
    """make_chain(13, layer_ms=1.0, ramp_ms=0.01): 12 sites n0..n11."""
    nodes = [f"n{i}" for i in range(13)]
    lat = {x: {1: 1.0} for x in nodes}
    ramp = {x: {1: 0.01} for x in nodes[:-1]}
    return ModelProfile(nodes, list(zip(nodes, nodes[1:])), lat, ramp, nodes[-1], name="chain")


def config4_window(n: int = 1_000_000, seed: int = 0) -> WindowArrays:
    """BASELINE config 4 window: agreement 0.5 -> 0.95 linear over n0..n11,
    continuity 0.9, miscalibration 0.05, 10 labels."""
    prof = config4_profile()
    sites = find_feasible_sites(prof)
    curve = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(sites)}
    return synthesize_window(prof, n, 0.9, curve, seed, miscalibration=0.05)
