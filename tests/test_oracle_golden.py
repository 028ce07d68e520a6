"""Pin the CPU oracle (oracle/) and the host-side modules to the reference.

Everything here runs without a GPU. The golden fixtures come from the
reference itself (tests/golden/make_golden.py, compiled backend).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import make_chain, make_record
from helpers import config4_curve, config4_profile, digest_records
from oracle import oracle as O
from paper_2312_05385_b200.engine import EEConfig, decision_scores, evaluate_record, serve_table
from paper_2312_05385_b200.graph import RampBudget, find_feasible_sites, initial_placement
from paper_2312_05385_b200.trace import synthesize_workload


def test_oracle_eval_matches_compiled_reference_bitwise(kernels_random):
    for w in kernels_random:
        acc, sav = O.eval_thresholds(w["scores"], w["cext"], w["serve"], float(w["vanilla"]), w["th"])
        assert np.array_equal(acc, w["acc"])
        assert np.array_equal(sav, w["sav"])  # same accumulation order as _exitcore.pyx
        np.testing.assert_allclose(sav, w["sav_numpy"], rtol=0, atol=1e-12)
        for row, want in zip(w["th"][:5], w["sites"]):
            assert np.array_equal(O.exit_sites(w["scores"], row), want)


def test_oracle_hist_consistent_with_eval(kernels_random):
    for w in kernels_random:
        hist, ok = O.eval_hist(w["scores"], w["cext"], w["th"])
        n = w["scores"].shape[0]
        assert (hist.sum(axis=1) == n).all()
        assert np.array_equal(ok / n, w["acc"])
        np.testing.assert_allclose(float(w["vanilla"]) - hist @ w["serve"] / n, w["sav"], atol=1e-12)


def test_oracle_edge_cases(golden):
    e = golden["edge"]
    s = np.array([[0.5, 0.1], [0.9, 0.9], [0.0, 0.9]])
    assert O.exit_sites(s, np.array([0.4, 0.2])).tolist() == e["semantics_sites"]
    s_nan = np.array([[np.nan, 0.1], [0.3, np.nan], [np.nan, np.nan], [0.2, 0.2]])
    assert O.exit_sites(s_nan, np.array([0.5, 0.5])).tolist() == e["nan_sites"]
    assert O.exit_sites(np.array([[0.5, 0.5]]), np.array([0.5, 0.6])).tolist() == e["tie_sites"]
    a, sv = O.eval_thresholds(np.zeros((4, 0)), np.ones((4, 1)), np.array([12.0]), 12.0,
                              np.zeros((3, 0)))
    assert [a.tolist(), sv.tolist()] == e["zero_ramps_compiled"]


def test_oracle_decision_scores(golden):
    e = golden["edge"]
    assert O.decision_scores(np.array([[0.8, 0.1, 0.3]]), 2).tolist() == e["decision_scores_k2"]
    errs = np.random.default_rng(e["decision_scores_rand_input_seed"]).random((64, 7))
    got = [x.hex() for x in O.decision_scores(errs, 3).ravel()]
    assert got == e["decision_scores_rand_k3_hex"]
    # the package's host twin agrees bit for bit
    assert [x.hex() for x in decision_scores(errs, 3).ravel()] == e["decision_scores_rand_k3_hex"]


def test_synthesizer_reproduces_reference_stream(golden):
    chain8 = make_chain(8)
    s8 = find_feasible_sites(chain8)
    curve8 = {x.position: 0.3 + 0.08 * i for i, x in enumerate(s8)}
    for seed, n, cont, mis in [(13, 64, 0.6, 0.25), (0, 300, 0.9, 0.05), (7, 200, 0.1, 0.4)]:
        w = synthesize_workload(chain8, n, cont, curve8, seed=seed, miscalibration=mis)
        assert digest_records(w.records) == golden["synth"][f"chain8_s{seed}_n{n}"]
    chain13 = config4_profile()
    s13 = find_feasible_sites(chain13)
    w13 = synthesize_workload(chain13, 2000, 0.9, config4_curve(s13), seed=0, miscalibration=0.05)
    assert digest_records(w13.records) == golden["synth"]["chain13_s0_n2000"]
    late = {x.position: 0.9 for x in s8}
    wl = synthesize_workload(chain8, 100, 0.5, curve8, seed=3, late_agreement_curve=late,
                             late_miscalibration=0.3, n_labels=2)
    assert digest_records(wl.records) == golden["synth"]["chain8_late_s3_n100_l2"]


def test_serve_tables_and_placement(golden):
    prof = make_chain(6, layer_ms=10.0, ramp_ms=0.5, batches=(1, 8, 32), batch_scale=0.1)
    sites = find_feasible_sites(prof)
    for b, want in golden["serves"].items():
        assert [x.hex() for x in serve_table(sites, prof, int(b))] == want
        assert [x.hex() for x in O.serve_table(sites, prof, int(b))] == want
    chain13 = config4_profile()
    s13 = find_feasible_sites(chain13)
    for f, want in golden["placement"].items():
        assert [x.position for x in initial_placement(s13, RampBudget(float(f)), chain13).sites] == want


def test_engine_known_answers(golden):
    chain4 = make_chain(4)
    sites = {x.position: x for x in find_feasible_sites(chain4)}
    rec = make_record(0, 0.0, {"n0": (0.5, 3), "n1": (0.2, 3), "n2": (0.9, 3)}, 3)
    out = evaluate_record(rec, EEConfig(((sites["n0"], 0.3), (sites["n1"], 0.8))), chain4)
    assert [out.exit_site, out.released_label, out.correct, out.serve_ms] == golden["edge"]["two_ramp_record"]
    recs = [
        make_record(0, 0, {"n0": (0.3, 1), "n1": (0.1, 1), "n2": (0.9, 1)}, 1),
        make_record(1, 1, {"n0": (0.5, 2), "n1": (0.5, 0), "n2": (0.9, 0)}, 0),
        make_record(2, 2, {"n0": (0.9, 5), "n1": (0.7, 5), "n2": (0.9, 5)}, 4),
        make_record(3, 3, {"n0": (0.2, 9), "n1": (0.0, 4), "n2": (0.9, 4)}, 4),
    ]
    active = [(sites["n0"], 0.4), (sites["n1"], 0.6)]
    acc, sav, rates = O.brute_window(recs, active, chain4)
    want = golden["edge"]["four_record"]
    assert acc == want[0] and sav == want[1] and rates == want[2]


def _tune_instance(entry):
    chain8 = make_chain(8)
    s8 = find_feasible_sites(chain8)
    w = synthesize_workload(chain8, 64, entry["continuity"], entry["curve"], seed=entry["seed"],
                            miscalibration=entry["miscal"])
    return chain8, [s8[1], s8[3], s8[5]], list(w.records)


def test_oracle_tune_matches_reference(golden):
    for entry in golden["tunes"]:
        prof, ramps, recs = _tune_instance(entry)
        th, sav, acc, rounds, evals, trace = O.tune(recs, ramps, prof)
        want = entry["tune"]
        assert th == [want["thresholds"][r.position] for r in ramps]
        assert sav.hex() == want["savings"]
        assert acc == want["accuracy"] and rounds == want["rounds"] and evals == want["evals"]
        assert [list(t) for t in trace] == want["trace"]
        for k in (2, 3):
            th, sav, *_ = O.tune(recs, ramps, prof, budget=0.05, k=k)
            assert th == [entry[f"tune_k{k}_b0.05"]["thresholds"][r.position] for r in ramps]
            assert sav.hex() == entry[f"tune_k{k}_b0.05"]["savings"]


def test_oracle_grid_matches_reference(golden):
    for entry in golden["tunes"][:4]:
        prof, ramps, recs = _tune_instance(entry)
        th, sav, acc, npts = O.grid_oracle(recs, ramps, prof, 0.01, 0.1)
        want = entry["grid_0.1"]
        assert th == [want["thresholds"][r.position] for r in ramps]
        assert sav.hex() == want["savings"] and acc == want["accuracy"] and npts == want["n_points"]


def test_reference_kernel_build_agrees_with_oracle(kernels_random):
    ref = O.reference_kernel()
    if ref is None:
        pytest.skip("oracle/_ref not built (run `make -C oracle ref` where /root/reference exists)")
    for w in kernels_random[:3]:
        acc, sav = ref.eval_thresholds(w["scores"], w["cext"], w["serve"], float(w["vanilla"]), w["th"])
        assert np.array_equal(acc, w["acc"]) and np.array_equal(sav, w["sav"])


def _config4_golden():
    import json
    import os

    from conftest import GOLDEN

    with open(os.path.join(GOLDEN, "config4_1m.json")) as fh:
        return json.load(fh)


def test_native_window_replay_equals_reference_generator_at_full_size():
    """The headline window (synth.config4_window: the native PCG64 replay,
    csrc/synth.cpp, host-only) equals the reference generator's 1M x 12 window
    packed by the reference's WindowEvaluator, byte for byte
    (tests/golden/make_config4_golden.py; trace.py:164-227, engine.py:152-163)."""
    import hashlib

    from paper_2312_05385_b200 import synth

    gold = _config4_golden()
    arrays = synth.config4_window(gold["n"])
    assert arrays.errs.shape == (gold["n"], gold["r"])
    assert hashlib.sha256(np.ascontiguousarray(arrays.errs).tobytes()).hexdigest() == gold["scores_sha256"]
    cext_u8 = np.ascontiguousarray(arrays.correct_ext().astype(np.uint8))
    assert hashlib.sha256(cext_u8.tobytes()).hexdigest() == gold["correct_u8_sha256"]
    prof = config4_profile()
    serve = serve_table(find_feasible_sites(prof), prof, 1)
    assert [x.hex() for x in serve] == gold["serve"]


def test_oracle_full_size_diagonal_matches_reference():
    """The C oracle on the full 1M x 12 window, all 64 diagonal candidates:
    acc bit-identical and sav bit-identical (same accumulation order) to the
    reference's compiled kernel."""
    from paper_2312_05385_b200 import synth

    gold = _config4_golden()
    arrays = synth.config4_window(gold["n"])
    prof = config4_profile()
    serve = serve_table(find_feasible_sites(prof), prof, 1)
    th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
    acc, sav = O.eval_thresholds(arrays.errs, arrays.correct_ext(), serve, prof.model_latency(1), th)
    assert [x.hex() for x in acc] == gold["diag_acc"]
    assert [x.hex() for x in sav] == gold["diag_sav"]
