"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference's golden vectors. Bit-exact for indices, histograms, accuracy
and — in exact mode — savings; histogram-mode savings within 1e-9 relative
(correctly rounded vs the reference's sequential sum)."""

from __future__ import annotations

import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN, make_chain
from helpers import axis_sweep, config4_curve, config4_profile, diagonal
from oracle import oracle as O
from paper_2312_05385_b200 import kernels
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import WindowArrays, synthesize_workload, window_arrays
from paper_2312_05385_b200.tuner import TunerParams, grid_oracle, tune

pytestmark = pytest.mark.gpu

SAV_RTOL = 1e-9  # histogram mode: correctly rounded total vs the reference's sequential fp64 sum


def random_window(rng, n, r, c, nan_frac=0.0, ties=False):
    scores = rng.random((n, r))
    if ties:
        scores = np.round(scores * 16) / 16
    if nan_frac:
        scores[rng.random((n, r)) < nan_frac] = np.nan
    cext = np.hstack([rng.integers(0, 2, size=(n, r)).astype(np.float64),
                      rng.integers(0, 2, size=(n, 1)).astype(np.float64)])
    serve = np.sort(rng.uniform(1.0, 50.0, size=r + 1))
    vanilla = float(serve[-1] + rng.uniform(0.0, 5.0))
    th = rng.random((c, r))
    if ties:
        th = np.round(th * 16) / 16
    return scores, cext, serve, vanilla, th


def check_hist(scores, cext, serve, vanilla, th, mode="hist"):
    acc, sav = kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode=mode)
    acc_o, sav_o = O.eval_thresholds(scores, cext, serve, vanilla, th)
    assert np.array_equal(acc, acc_o)
    np.testing.assert_allclose(sav, sav_o, rtol=SAV_RTOL, atol=1e-12)
    return acc, sav


def test_golden_random_windows_exact_bitwise(cuda, kernels_random):
    for w in kernels_random:
        acc, sav = kernels.eval_thresholds(w["scores"], w["cext"], w["serve"], float(w["vanilla"]),
                                           w["th"])
        assert np.array_equal(acc, w["acc"]) and np.array_equal(sav, w["sav"])
        for row, want in zip(w["th"][:5], w["sites"]):
            assert np.array_equal(kernels.exit_sites(w["scores"], row), want)


def test_golden_random_windows_hist_mode(cuda, kernels_random):
    for w in kernels_random:
        acc, sav = kernels.eval_thresholds(w["scores"], w["cext"], w["serve"], float(w["vanilla"]),
                                           w["th"], mode="hist")
        assert np.array_equal(acc, w["acc"])
        np.testing.assert_allclose(sav, w["sav"], rtol=0, atol=1e-12)


def test_edge_semantics(cuda, golden):
    e = golden["edge"]
    s = np.array([[0.5, 0.1], [0.9, 0.9], [0.0, 0.9]])
    assert kernels.exit_sites(s, np.array([0.4, 0.2])).tolist() == e["semantics_sites"]
    s_nan = np.array([[np.nan, 0.1], [0.3, np.nan], [np.nan, np.nan], [0.2, 0.2]])
    assert kernels.exit_sites(s_nan, np.array([0.5, 0.5])).tolist() == e["nan_sites"]
    assert kernels.exit_sites(np.array([[0.5, 0.5]]), np.array([0.5, 0.6])).tolist() == e["tie_sites"]
    a, sv = kernels.eval_thresholds(np.zeros((4, 0)), np.ones((4, 1)), np.array([12.0]), 12.0,
                                    np.zeros((3, 0)))
    assert [a.tolist(), sv.tolist()] == e["zero_ramps_compiled"]
    a, sv = kernels.eval_thresholds(np.zeros((0, 2)), np.ones((0, 3)), np.ones(3), 1.0,
                                    np.zeros((2, 2)))
    assert np.isnan(a).all() and np.isnan(sv).all()
    a, sv = kernels.eval_thresholds(np.zeros((2, 2)), np.ones((2, 3)), np.ones(3), 1.0,
                                    np.zeros((0, 2)))
    assert a.shape == (0,) and sv.shape == (0,)
    assert kernels.exit_sites(np.zeros((3, 0)), np.zeros(0)).tolist() == [0, 0, 0]


def test_nan_ties_and_signed_zero_both_modes(cuda):
    rng = np.random.default_rng(11)
    for mode in ("exact", "hist"):
        scores, cext, serve, vanilla, th = random_window(rng, 3001, 5, 70, nan_frac=0.05, ties=True)
        th[3, 2] = np.nan  # NaN threshold never exits
        th[4, :] = -0.0
        scores[:10, 0] = 0.0
        th[5, 0] = np.inf
        scores[10:20, 1] = -np.inf
        check_hist(scores, cext, serve, vanilla, th, mode=mode)
        for row in th[:8]:
            assert np.array_equal(kernels.exit_sites(scores, row), O.exit_sites(scores, row))


def test_not_binary_correct_ext_is_rejected(cuda):
    scores = np.zeros((4, 2))
    cext = np.ones((4, 3))
    cext[1, 1] = 0.5
    with pytest.raises(ValueError, match="0.0 and 1.0"):
        kernels.eval_thresholds(scores, cext, np.ones(3), 1.0, np.zeros((1, 2)))


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 8, 12, 13, 16, 17, 24, 31])
def test_hist_histograms_exact_across_ramp_counts(cuda, r):
    rng = np.random.default_rng(100 + r)
    n = 5000 + 37 * r  # not a multiple of the 256-sample tile
    scores, cext, serve, vanilla, th = random_window(rng, n, r, 150, ties=(r % 2 == 0))
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    hist, ok = ev.histograms(th)
    hist_o, ok_o = O.eval_hist(scores, cext, th)
    assert np.array_equal(hist, hist_o) and np.array_equal(ok, ok_o)
    check_hist(scores, cext, serve, vanilla, th)


def test_more_than_127_distinct_thresholds_per_ramp(cuda):
    rng = np.random.default_rng(3)
    scores, cext, serve, vanilla, th = random_window(rng, 8000, 6, 700)  # forces several chunks
    check_hist(scores, cext, serve, vanilla, th)


def test_exact_mode_bitwise_vs_oracle_large_grid(cuda):
    rng = np.random.default_rng(4)
    scores, cext, serve, vanilla, th = random_window(rng, 64, 3, 20000)
    acc, sav = kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode="exact")
    acc_o, sav_o = O.eval_thresholds(scores, cext, serve, vanilla, th)
    assert np.array_equal(acc, acc_o) and np.array_equal(sav, sav_o)


def test_exact_mode_long_window_bitwise(cuda):
    rng = np.random.default_rng(6)
    scores, cext, serve, vanilla, th = random_window(rng, 20000, 12, 7)
    acc, sav = kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode="exact")
    acc_o, sav_o = O.eval_thresholds(scores, cext, serve, vanilla, th)
    assert np.array_equal(acc, acc_o) and np.array_equal(sav, sav_o)


def test_device_decision_scores_bitwise(cuda, golden):
    e = golden["edge"]
    errs = np.random.default_rng(e["decision_scores_rand_input_seed"]).random((64, 7))
    prof = make_chain(8)
    arrays = WindowArrays(errs, np.ones((64, 8), dtype=np.uint8))
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:7], prof, k=3)
    assert [x.hex() for x in ev.scores.ravel()] == e["decision_scores_rand_k3_hex"]


def _tune_case(entry):
    chain8 = make_chain(8)
    s8 = find_feasible_sites(chain8)
    w = synthesize_workload(chain8, 64, entry["continuity"], entry["curve"], seed=entry["seed"],
                            miscalibration=entry["miscal"])
    return chain8, [s8[1], s8[3], s8[5]], list(w.records)


@pytest.mark.parametrize("device_loop", [True, False])
def test_tune_matches_reference_bitwise(cuda, golden, device_loop):
    for entry in golden["tunes"]:
        prof, ramps, recs = _tune_case(entry)
        res = tune(recs, ramps, TunerParams(), prof, device_loop=device_loop)
        want = entry["tune"]
        assert dict(res.thresholds) == want["thresholds"]
        assert res.savings_ms.hex() == want["savings"]
        assert res.accuracy == want["accuracy"]
        assert (res.rounds, res.evals) == (want["rounds"], want["evals"])
        assert [list(t) for t in res.step_trace] == want["trace"]
        for k in (2, 3):
            rk = tune(recs, ramps, TunerParams(acc_loss_budget=0.05), prof, k=k,
                      device_loop=device_loop)
            assert dict(rk.thresholds) == entry[f"tune_k{k}_b0.05"]["thresholds"]
            assert rk.savings_ms.hex() == entry[f"tune_k{k}_b0.05"]["savings"]


def test_grid_oracle_matches_reference_bitwise(cuda, golden):
    for entry in golden["tunes"]:
        prof, ramps, recs = _tune_case(entry)
        for key, step in (("grid_0.1", 0.1), ("grid_0.01", 0.01)):
            if key not in entry:
                continue
            res = grid_oracle(recs, ramps, 0.01, step, prof)
            want = entry[key]
            assert dict(res.thresholds) == want["thresholds"]
            assert res.savings_ms.hex() == want["savings"]
            assert res.accuracy == want["accuracy"] and res.n_points == want["n_points"]


@pytest.mark.parametrize("device_loop", [True, False])
def test_tune_config1_window(cuda, golden, device_loop):
    chain13 = config4_profile()
    s13 = find_feasible_sites(chain13)
    w = synthesize_workload(chain13, 1000, 0.7, config4_curve(s13), seed=42, miscalibration=0.1)
    ramps = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
    res = tune(list(w.records), ramps, TunerParams(), chain13, device_loop=device_loop)
    want = golden["tune_1k"]
    assert dict(res.thresholds) == want["thresholds"]
    assert res.savings_ms.hex() == want["savings"]
    assert (res.accuracy, res.rounds, res.evals) == (want["accuracy"], want["rounds"], want["evals"])


@pytest.mark.parametrize("r,n", [(12, 600), (12, 3000), (12, 20000), (20, 600), (20, 3000),
                                 (31, 600), (31, 3000), (31, 20000)])
def test_tune_kernel_variants_match_exact_host_loop_and_oracle(cuda, r, n):
    """Every k_tune variant (R <= 8 / 16 / 32 register buckets) and every
    shared-memory layout branch (window in shared or global memory, addend rows
    in shared or global memory) against the exact host loop and the Python
    Algorithm 1 over the C oracle kernel (tuner.py:97-171): bit-identical."""
    prof = make_chain(r + 1, layer_ms=1.0, ramp_ms=0.01)
    sites = find_feasible_sites(prof)
    curve = {x.position: 0.4 + 0.5 * i / max(1, r - 1) for i, x in enumerate(sites)}
    w = synthesize_workload(prof, n, 0.8, curve, seed=1000 + r + n, miscalibration=0.1)
    recs = list(w.records)
    ev = WindowEvaluator(recs, sites, prof, mode="hist")  # hist: the host loop must still score exactly
    dev = tune(recs, sites, TunerParams(), prof, evaluator=ev, device_loop=True)
    host = tune(recs, sites, TunerParams(), prof, evaluator=ev, device_loop=False)
    assert dev.thresholds == host.thresholds
    assert dev.savings_ms.hex() == host.savings_ms.hex()
    assert (dev.accuracy, dev.rounds, dev.evals) == (host.accuracy, host.rounds, host.evals)
    th, sav, acc, rounds, evals, _ = O.tune(recs, sites, prof)
    assert [dev.thresholds[x.position] for x in sites] == list(th)
    assert dev.savings_ms.hex() == float(sav).hex() and dev.accuracy == acc
    assert (dev.rounds, dev.evals) == (rounds, evals)


def test_tune_rejects_mismatched_evaluator(cuda):
    prof = make_chain(5)
    sites = find_feasible_sites(prof)
    w = synthesize_workload(prof, 64, 0.5, {x.position: 0.7 for x in sites}, seed=3)
    ev = WindowEvaluator(list(w.records), sites[:3], prof)
    with pytest.raises(Exception, match="evaluator window covers sites"):
        tune(list(w.records), sites, TunerParams(), prof, evaluator=ev)


def test_estimate_utilities_golden(cuda, golden):
    from conftest import make_record
    from paper_2312_05385_b200.engine import EEConfig
    from paper_2312_05385_b200.ramps import estimate_utilities

    chain4 = make_chain(4)
    sites = {x.position: x for x in find_feasible_sites(chain4)}
    recs = [
        make_record(0, 0, {"n0": (0.3, 1), "n1": (0.1, 1), "n2": (0.9, 1)}, 1),
        make_record(1, 1, {"n0": (0.5, 2), "n1": (0.5, 0), "n2": (0.9, 0)}, 0),
        make_record(2, 2, {"n0": (0.9, 5), "n1": (0.7, 5), "n2": (0.9, 5)}, 4),
        make_record(3, 3, {"n0": (0.2, 9), "n1": (0.0, 4), "n2": (0.9, 4)}, 4),
    ]
    cfg = EEConfig(((sites["n0"], 0.4), (sites["n1"], 0.6)))
    assert estimate_utilities(recs, cfg, chain4).to_dict() == golden["edge"]["utilities"]


def test_medium_sweep_window_against_reference(cuda):
    gold = np.load(os.path.join(GOLDEN, "sweep_medium.npz"))
    chain13 = config4_profile()
    s13 = find_feasible_sites(chain13)
    w = synthesize_workload(chain13, 5000, 0.9, config4_curve(s13), seed=0, miscalibration=0.05)
    arrays = window_arrays(w.records, s13)
    for mode in ("exact", "hist"):
        ev = WindowEvaluator.from_arrays(arrays, s13, chain13, mode=mode)
        assert np.array_equal(ev.serve, gold["serve"])
        for fam, th in (("diag", diagonal()), ("axis", axis_sweep())):
            acc, sav = ev.evaluate_many(th)
            assert np.array_equal(acc, gold[f"{fam}_acc"])
            if mode == "exact":
                assert np.array_equal(sav, gold[f"{fam}_sav"])
            else:
                np.testing.assert_allclose(sav, gold[f"{fam}_sav"], rtol=SAV_RTOL, atol=0)


def _config4_golden():
    with open(os.path.join(GOLDEN, "config4_1m.json")) as fh:
        return json.load(fh)


def _unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def test_full_size_config4_histograms(cuda):
    """1M x 12 at full size, ALL 64 diagonal candidates: exact histograms and
    correct counts against the C oracle, acc bit-identical and sav within
    1e-9 * vanilla of the REFERENCE's own compiled kernel on the reference's own
    window (tests/golden/config4_1m.json), plus size-independent invariants."""
    from paper_2312_05385_b200 import synth

    gold = _config4_golden()
    prof = config4_profile()
    sites = find_feasible_sites(prof)
    arrays = synth.config4_window(1_000_000)
    assert hashlib.sha256(np.ascontiguousarray(arrays.errs).tobytes()).hexdigest() == gold["scores_sha256"]
    ev = WindowEvaluator.from_arrays(arrays, sites, prof, mode="hist")
    assert [x.hex() for x in ev.serve] == gold["serve"]
    th = diagonal()
    hist, ok = ev.histograms(th)
    n = arrays.n
    assert (hist.sum(axis=1) == n).all()
    # raising every threshold never delays an exit: exits at ramp 0 are monotone
    assert (np.diff(hist[:, 0]) >= 0).all()
    cext = arrays.correct_ext()
    hist_o, ok_o = O.eval_hist(arrays.errs, cext, th)
    assert np.array_equal(hist, hist_o) and np.array_equal(ok, ok_o)
    acc, sav = ev.evaluate_many(th)
    assert np.array_equal(acc, _unhex(gold["diag_acc"]))
    # sav is a difference of O(vanilla) quantities: compare on the serve-time scale
    np.testing.assert_allclose(sav, _unhex(gold["diag_sav"]), rtol=0, atol=1e-9 * ev.vanilla_ms)
    # and our value is the correctly rounded mean (within 2 ulp of the exact rational)
    for row, s_got in zip(hist, sav):
        exact = Fraction(ev.vanilla_ms) - sum(int(k) * Fraction(float(v)) for k, v in zip(row, ev.serve)) / n
        assert abs(Fraction(s_got) - exact) <= 2 * np.spacing(abs(float(exact)))


def test_full_size_config4_axis_family_vs_reference(cuda):
    """The 768-row axis family over the full 1M x 12 window: acc
    bit-identical to the reference's compiled kernel, sav within 1e-9 * vanilla."""
    from paper_2312_05385_b200 import kernels as K
    from paper_2312_05385_b200 import synth

    gold = _config4_golden()
    prof = config4_profile()
    sites = find_feasible_sites(prof)
    ev = WindowEvaluator.from_arrays(synth.config4_window(1_000_000), sites, prof, mode="hist")
    axis = np.full((768, 12), 0.3)
    for j in range(12):
        axis[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
    assert K.classify_candidates(axis)[0] == "axis"
    acc, sav = ev.evaluate_many(axis)
    assert np.array_equal(acc, _unhex(gold["axis_acc"]))
    np.testing.assert_allclose(sav, _unhex(gold["axis_sav"]), rtol=0, atol=1e-9 * ev.vanilla_ms)


@pytest.mark.parametrize("r,clustered", [(1, False), (3, True), (7, False), (12, False),
                                         (12, True), (16, False), (31, True)])
def test_diagonal_family_path_matches_generic(cuda, r, clustered):
    """The single-pass diagonal kernel and the generic SWAR kernel agree exactly
    (clustered thresholds exercise the multi-threshold-per-bin scan)."""
    from paper_2312_05385_b200 import _native

    rng = np.random.default_rng(700 + r)
    n = 20000 + 3 * r
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1, nan_frac=0.02, ties=(r % 2 == 1))
    extra = [0.0, -0.0, np.inf, -np.inf, np.nan]
    if clustered:
        extra += [0.5 + k * 1e-13 for k in range(5)]
        scores[:50, 0] = 0.5 + 2e-13
    vals = np.concatenate([np.round(rng.random(90) * 32) / 32, extra])
    rng.shuffle(vals)
    th = np.repeat(vals[:, None], r, axis=1)
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    hist_d, ok_d = ev.histograms(th)
    acc_d, sav_d = ev.evaluate_many(th)
    _native.set_special(False)
    try:
        hist_g, ok_g = ev.histograms(th)
        acc_g, sav_g = ev.evaluate_many(th)
    finally:
        _native.set_special(True)
    assert np.array_equal(hist_d, hist_g) and np.array_equal(ok_d, ok_g)
    assert np.array_equal(acc_d, acc_g) and np.array_equal(sav_d, sav_g)
    hist_o, ok_o = O.eval_hist(scores, cext, th)
    assert np.array_equal(hist_d, hist_o) and np.array_equal(ok_d, ok_o)


@pytest.mark.parametrize("r,n,nan_base", [(2, 37, False), (6, 5003, True), (12, 40001, False),
                                          (12, 70001, True), (16, 20011, False)])
def test_axis_family_path_matches_generic_and_oracle(cuda, r, n, nan_base):
    """k_axis (rows = a base vector with one coordinate swept over a shared value
    set, SURVEY 8(d)'s C = 768 family) against the generic SWAR kernel and the C
    oracle: ragged tails, NaN/inf/-0 scores, NaN and +-inf values, rows equal to
    the base, a NaN base entry, no-exit bit 0 rows; the k_axis launch is checked."""
    from paper_2312_05385_b200 import _native

    rng = np.random.default_rng(4400 + r + n)
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1, nan_frac=0.01)
    scores[rng.random((n, r)) < 0.01] = np.inf
    scores[rng.random((n, r)) < 0.01] = -0.0
    scores[rng.random((n, r)) < 0.02] = 0.3  # ties with the base
    cext[:, r] = (rng.random(n) < 0.8).astype(np.float64)
    vals = np.concatenate([np.arange(60) / 59.0, [np.inf, -np.inf, -0.0, np.nan]])
    base = np.full(r, 0.3)
    if nan_base:
        base[r // 2] = np.nan
    rows = [base.copy()] if r < 16 else []  # a row equal to the base (C <= 1024)
    for j in range(r):
        for v in vals:
            row = base.copy()
            row[j] = v
            rows.append(row)
    th = np.array(rows)
    rng.shuffle(th)
    assert th.shape[0] <= 1024
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    _native.profile_read()
    _native.profile_enable(True)
    try:
        hist_a, ok_a = ev.histograms(th)
        acc_a, sav_a = ev.evaluate_many(th)
    finally:
        _native.profile_enable(False)
    assert "k_axis" in _native.profile_read()
    _native.set_special(False)
    try:
        hist_g, ok_g = ev.histograms(th)
        acc_g, sav_g = ev.evaluate_many(th)
    finally:
        _native.set_special(True)
    assert np.array_equal(hist_a, hist_g) and np.array_equal(ok_a, ok_g)
    assert np.array_equal(acc_a, acc_g) and np.array_equal(sav_a, sav_g)
    hist_o, ok_o = O.eval_hist(scores, cext, th)
    assert np.array_equal(hist_a, hist_o) and np.array_equal(ok_a, ok_o)
    # repeated call: the totals are rebuilt from zero
    hist2, ok2 = ev.histograms(th)
    assert np.array_equal(hist2, hist_a) and np.array_equal(ok2, ok_a)


@pytest.mark.parametrize("r,n,nwin", [(12, 40001, 5), (2, 33, 3), (16, 100003, 7), (6, 4099, 1), (8, 1, 2)])
def test_windows_batch_matches_per_window_sweeps(cuda, r, n, nwin):
    """ee_eval_thresholds_windows (k_diag3_windows_db: one persistent sweep over
    several resident windows, folds overlapped by dedicated warps, + one
    finalisation) returns, per window, the bits a per-window sweep returns;
    windows repeated in the order are independent results. Ragged tails, tiny
    windows (fewer chunks than stream warps), every even R up to 16, odd window
    counts (both cell buffers in turn)."""
    import torch

    from paper_2312_05385_b200 import kernels as K

    prof = make_chain(r + 1)
    sites = find_feasible_sites(prof)[:r]
    evs = []
    for w in range(3):
        rng = np.random.default_rng(6100 + w)
        scores, cext, *_ = random_window(rng, n, r, 1, nan_frac=0.01)
        cext[:, r] = (rng.random(n) < 0.8).astype(np.float64)
        evs.append(WindowEvaluator.from_arrays(WindowArrays(scores, cext.astype(np.uint8)), sites, prof,
                                               mode="hist"))
    vals = np.concatenate([np.arange(60) / 59.0, [np.nan, -np.inf]])
    th = np.repeat(vals[:, None], r, axis=1)
    order = [(2 * i + 1) % 3 for i in range(nwin)]  # 1, 0, 2, 1, 0, ...
    acc, sav = K.eval_thresholds_windows(evs, th, order)
    torch.cuda.synchronize()
    for row, wi in enumerate(order):
        a1, s1 = evs[wi].evaluate_many(th)
        assert np.array_equal(acc[row].cpu().numpy(), a1)
        assert np.array_equal(sav[row].cpu().numpy(), s1)


@pytest.mark.parametrize("r,n", [(5, 3001), (12, 1), (12, 31), (4, 64)])
def test_axis_family_edges_and_fallback(cuda, r, n):
    """Single-coordinate rows outside k_axis's envelope (odd R) take the generic
    path; tiny windows (n < one chunk per CTA) run k_axis; all exact vs the oracle."""
    from paper_2312_05385_b200 import _native

    rng = np.random.default_rng(8800 + r + n)
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1, nan_frac=0.02)
    th = np.full((1 + r * 20, r), 0.45)
    for j in range(r):
        th[1 + j * 20:1 + (j + 1) * 20, j] = np.arange(20) / 19.0
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    _native.profile_read()
    _native.profile_enable(True)
    try:
        hist, ok = ev.histograms(th)
        acc, sav = ev.evaluate_many(th)
    finally:
        _native.profile_enable(False)
    launched = _native.profile_read()
    assert ("k_axis" in launched) == (r % 2 == 0), launched
    hist_o, ok_o = O.eval_hist(scores, cext, th)
    assert np.array_equal(hist, hist_o) and np.array_equal(ok, ok_o)
    acc_o, sav_o = O.eval_thresholds(scores, cext, ev.serve, ev.vanilla_ms, th)
    assert np.array_equal(acc, acc_o)
    np.testing.assert_allclose(sav, sav_o, rtol=SAV_RTOL, atol=1e-12)


@pytest.mark.parametrize("r,n,m,c_rep", [(2, 1, 5, 1), (4, 31, 17, 1), (6, 33, 64, 1),
                                         (10, 4099, 127, 1), (12, 70001, 64, 1), (12, 2500, 40, 20),
                                         (14, 9000, 100, 1), (16, 12345, 126, 2)])
def test_diag2_matches_diag1_and_oracle(cuda, r, n, m, c_rep):
    """k_diag3 (lane-private cumulative counters, m <= 64) and k_diag2
    (coalesced, replicated bin table, one launch) against k_diag and the C
    oracle: ragged tails (n % 32 != 0), up to 127 distinct thresholds incl.
    +-inf and +-0, NaN rows and NaN scores, rows whose no-exit bit is 0, and
    more than 512 candidates (device position map)."""
    from paper_2312_05385_b200 import _native

    rng = np.random.default_rng(9100 + r + n)
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1, nan_frac=0.01)
    scores[rng.random((n, r)) < 0.01] = np.inf
    scores[rng.random((n, r)) < 0.01] = -0.0
    cext[:, r] = (rng.random(n) < 0.8).astype(np.float64)  # some samples with bit r = 0
    extra = np.array([0.0, np.inf, -np.inf, 1.0])
    vals = np.unique(np.concatenate([np.round(rng.random(4 * m) * 997) / 997, extra]))[:m]
    rows = np.concatenate([vals, [np.nan]])
    rows = np.repeat(rows, c_rep)
    rng.shuffle(rows)
    th = np.repeat(rows[:, None], r, axis=1)
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    hist2, ok2 = ev.histograms(th)
    acc2, sav2 = ev.evaluate_many(th)
    for ver in (6, 5, 2, 1):
        _native.set_diag_version(ver)
        try:
            hist1, ok1 = ev.histograms(th)
            acc1, sav1 = ev.evaluate_many(th)
        finally:
            _native.set_diag_version()
        assert np.array_equal(hist2, hist1) and np.array_equal(ok2, ok1), ver
        assert np.array_equal(acc2, acc1) and np.array_equal(sav2, sav1), ver
    hist_o, ok_o = O.eval_hist(scores, cext, th)
    assert np.array_equal(hist2, hist_o) and np.array_equal(ok2, ok_o)
    # repeated calls on the same workspace: the accumulator is left zeroed
    hist3, ok3 = ev.histograms(th)
    assert np.array_equal(hist3, hist2) and np.array_equal(ok3, ok2)
