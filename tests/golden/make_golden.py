"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (the reference is only present in the build container):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory under /tmp (the
reference tree is read-only and its Cython build writes in-tree), builds the
compiled backend, asserts `eesim._kernels.BACKEND == "compiled"` and records
inputs/outputs of the functions on the exit-decision path. Nothing here is
imported at test time; tests read the fixture files only.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
SCRATCH = "/tmp/eeb200_golden_ref"


def load_reference():
    if not os.path.isdir(os.path.join(SCRATCH, "src", "eesim")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree(REF_PKG, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, os.path.join(SCRATCH, "tests"))
    import eesim._kernels as K

    assert K.BACKEND == "compiled", K.BACKEND
    return K


def digest_records(records) -> str:
    h = hashlib.sha256()
    for rec in records:
        obj = {"id": rec.id, "a": rec.arrival_ms, "f": rec.final_label,
               "s": {k: [v.err.hex(), v.label] for k, v in sorted(rec.ramp_signals.items())}}
        h.update(json.dumps(obj, sort_keys=True).encode())
    return h.hexdigest()


def main():
    K = load_reference()
    from conftest import make_chain, make_record  # reference test helpers
    from eesim.engine import EEConfig, WindowEvaluator, decision_scores, evaluate_record, evaluate_window
    from eesim.graph import RampBudget, find_feasible_sites, initial_placement
    from eesim.ramps import estimate_utilities
    from eesim.trace import synthesize_workload
    from eesim.tuner import TunerParams, grid_oracle, tune

    cy = K.get_backend("compiled")
    py = K.get_backend("python")

    # 1. test_kernels.random_window stream (pkg/tests/test_kernels.py:7-15,26-45)
    rng = np.random.default_rng(99)
    arrays = {}
    for w in range(10):
        n, r, c = 40, 3, 50
        scores = rng.random((n, r))
        cext = np.hstack([rng.integers(0, 2, size=(n, r)).astype(np.float64), np.ones((n, 1))])
        serve = np.sort(rng.uniform(1.0, 50.0, size=r + 1))
        vanilla = float(serve[-1] + rng.uniform(0.0, 5.0))
        th = rng.random((c, r))
        acc, sav = cy.eval_thresholds(scores, cext, serve, vanilla, th)
        acc_p, sav_p = py.eval_thresholds(scores, cext, serve, vanilla, th)
        sites = np.stack([cy.exit_sites(scores, np.ascontiguousarray(row)) for row in th[:5]])
        for key, val in dict(scores=scores, cext=cext, serve=serve, vanilla=np.array(vanilla),
                             th=th, acc=acc, sav=sav, acc_numpy=acc_p, sav_numpy=sav_p,
                             sites=sites).items():
            arrays[f"w{w}_{key}"] = val
    np.savez_compressed(os.path.join(HERE, "kernels_random.npz"), **arrays)

    # 2. edge cases of the seam (_ref.py:49-52, _exitcore.pyx) incl. NaN and ties
    edge = {}
    s = np.array([[0.5, 0.1], [0.9, 0.9], [0.0, 0.9]])
    edge["semantics_sites"] = cy.exit_sites(s, np.array([0.4, 0.2])).tolist()
    s_nan = np.array([[np.nan, 0.1], [0.3, np.nan], [np.nan, np.nan], [0.2, 0.2]])
    edge["nan_sites"] = cy.exit_sites(s_nan, np.array([0.5, 0.5])).tolist()
    edge["tie_sites"] = cy.exit_sites(np.array([[0.5, 0.5]]), np.array([0.5, 0.6])).tolist()
    a, sv = cy.eval_thresholds(np.zeros((4, 0)), np.ones((4, 1)), np.array([12.0]), 12.0,
                               np.zeros((3, 0)))
    edge["zero_ramps_compiled"] = [a.tolist(), sv.tolist()]
    a, sv = cy.eval_thresholds(np.zeros((0, 2)), np.ones((0, 3)), np.ones(3), 1.0, np.zeros((2, 2)))
    edge["empty_window_compiled"] = [[str(x) for x in a], [str(x) for x in sv]]
    edge["decision_scores_k2"] = decision_scores(np.array([[0.8, 0.1, 0.3]]), k=2).tolist()
    rng = np.random.default_rng(5)
    errs = rng.random((64, 7))
    edge["decision_scores_rand_k3_hex"] = [x.hex() for x in decision_scores(errs, 3).ravel()]
    edge["decision_scores_rand_input_seed"] = 5

    # 3. engine known answers (pkg/tests/test_engine.py:45-111)
    chain4 = make_chain(4)
    sites4 = {x.position: x for x in find_feasible_sites(chain4)}
    cfg = EEConfig(((sites4["n0"], 0.4), (sites4["n1"], 0.6)))
    recs = [
        make_record(0, 0, {"n0": (0.3, 1), "n1": (0.1, 1), "n2": (0.9, 1)}, 1),
        make_record(1, 1, {"n0": (0.5, 2), "n1": (0.5, 0), "n2": (0.9, 0)}, 0),
        make_record(2, 2, {"n0": (0.9, 5), "n1": (0.7, 5), "n2": (0.9, 5)}, 4),
        make_record(3, 3, {"n0": (0.2, 9), "n1": (0.0, 4), "n2": (0.9, 4)}, 4),
    ]
    st = evaluate_window(recs, cfg, chain4)
    edge["four_record"] = [st.accuracy, st.mean_savings_ms, dict(st.exit_rates)]
    out = evaluate_record(make_record(0, 0.0, {"n0": (0.5, 3), "n1": (0.2, 3), "n2": (0.9, 3)}, 3),
                          EEConfig(((sites4["n0"], 0.3), (sites4["n1"], 0.8))), chain4)
    edge["two_ramp_record"] = [out.exit_site, out.released_label, out.correct, out.serve_ms]
    util = estimate_utilities(recs, cfg, chain4)
    edge["utilities"] = util.to_dict()

    # 4. synthesize_workload stream digests (trace.py:164-227)
    synth = {}
    chain8 = make_chain(8)
    s8 = find_feasible_sites(chain8)
    curve8 = {x.position: 0.3 + 0.08 * i for i, x in enumerate(s8)}
    for seed, n, cont, mis in [(13, 64, 0.6, 0.25), (0, 300, 0.9, 0.05), (7, 200, 0.1, 0.4)]:
        w = synthesize_workload(chain8, n, cont, curve8, seed=seed, miscalibration=mis)
        synth[f"chain8_s{seed}_n{n}"] = digest_records(w.records)
    chain13 = make_chain(13, layer_ms=1.0, ramp_ms=0.01)
    s13 = find_feasible_sites(chain13)
    curve13 = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(s13)}
    w13 = synthesize_workload(chain13, 2000, 0.9, curve13, seed=0, miscalibration=0.05)
    synth["chain13_s0_n2000"] = digest_records(w13.records)
    late = {x.position: 0.9 for x in s8}
    wl = synthesize_workload(chain8, 100, 0.5, curve8, seed=3, late_agreement_curve=late,
                             late_miscalibration=0.3, n_labels=2)
    synth["chain8_late_s3_n100_l2"] = digest_records(wl.records)

    # 5. serve tables and placement (engine.py:124-132, graph.py:303-325)
    prof_b = make_chain(6, layer_ms=10.0, ramp_ms=0.5, batches=(1, 8, 32), batch_scale=0.1)
    sb = find_feasible_sites(prof_b)
    from eesim.engine import _serve_table

    serves = {str(b): [x.hex() for x in _serve_table(sb, prof_b, b)] for b in (1, 5, 8, 20, 32, 64)}
    placement = {str(f): [x.position for x in initial_placement(s13, RampBudget(f), chain13).sites]
                 for f in (0.0, 0.001, 0.02, 0.05, 0.2)}

    # 6. tune / grid on the acceptance instances (test_acceptance.py:56-85)
    tunes = []
    rng = np.random.default_rng(2024)
    ramps = [s8[1], s8[3], s8[5]]
    for seed in range(12):
        lo = float(rng.uniform(0.2, 0.5))
        hi = float(rng.uniform(lo, 0.95))
        curve = {x.position: lo + (hi - lo) * i / 6 for i, x in enumerate(s8)}
        cont = float(rng.uniform(0, 1))
        mis = float(rng.uniform(0, 0.4))
        w = synthesize_workload(chain8, 64, cont, curve, seed=seed, miscalibration=mis)
        res = tune(list(w.records), ramps, TunerParams(), chain8)
        entry = {"seed": seed, "curve": curve, "continuity": cont, "miscal": mis,
                 "tune": {"thresholds": dict(res.thresholds), "savings": res.savings_ms.hex(),
                          "accuracy": res.accuracy, "rounds": res.rounds, "evals": res.evals,
                          "trace": [list(t) for t in res.step_trace]}}
        g1 = grid_oracle(list(w.records), ramps, 0.01, 0.1, chain8)
        entry["grid_0.1"] = {"thresholds": dict(g1.thresholds), "savings": g1.savings_ms.hex(),
                             "accuracy": g1.accuracy, "n_points": g1.n_points}
        if seed < 3:
            g2 = grid_oracle(list(w.records), ramps, 0.01, 0.01, chain8)
            entry["grid_0.01"] = {"thresholds": dict(g2.thresholds),
                                  "savings": g2.savings_ms.hex(), "accuracy": g2.accuracy,
                                  "n_points": g2.n_points}
        for k in (2, 3):
            rk = tune(list(w.records), ramps, TunerParams(acc_loss_budget=0.05), chain8, k=k)
            entry[f"tune_k{k}_b0.05"] = {"thresholds": dict(rk.thresholds),
                                         "savings": rk.savings_ms.hex(), "rounds": rk.rounds}
        tunes.append(entry)
    # a config-1 sized window: 1000 records x 6 ramps
    w1k = synthesize_workload(chain13, 1000, 0.7, curve13, seed=42, miscalibration=0.1)
    r6 = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
    res = tune(list(w1k.records), r6, TunerParams(), chain13)
    tune_1k = {"thresholds": dict(res.thresholds), "savings": res.savings_ms.hex(),
               "accuracy": res.accuracy, "rounds": res.rounds, "evals": res.evals}

    # 7. medium sweep window (config-4 generator, 5000 records): diagonal C=64
    w5k = synthesize_workload(chain13, 5000, 0.9, curve13, seed=0, miscalibration=0.05)
    ev = WindowEvaluator(list(w5k.records), s13, chain13)
    diag = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
    acc, sav = ev.evaluate_many(diag)
    axis = np.full((768, 12), 0.3)
    for j in range(12):
        axis[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
    acc_ax, sav_ax = ev.evaluate_many(axis)
    np.savez_compressed(os.path.join(HERE, "sweep_medium.npz"), diag_acc=acc, diag_sav=sav,
                        axis_acc=acc_ax, axis_sav=sav_ax,
                        serve=ev.serve, vanilla=np.array(ev.vanilla_ms),
                        scores_sha=np.array(hashlib.sha256(ev.scores.tobytes()).hexdigest()))

    doc = {"edge": edge, "synth": synth, "serves": serves, "placement": placement,
           "tunes": tunes, "tune_1k": tune_1k,
           "generated_by": "tests/golden/make_golden.py from /root/reference/pkg (compiled backend)"}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    print("wrote", HERE)


if __name__ == "__main__":
    main()
