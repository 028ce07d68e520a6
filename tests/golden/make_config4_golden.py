"""Golden fixture for the full-size config-4 window, from the REFERENCE itself.

    python tests/golden/make_config4_golden.py

Builds BASELINE config 4's window (1M records x 12 ramps) with the reference's
own generator and packing — eesim.trace.synthesize_workload (trace.py:164-227)
and eesim.engine.WindowEvaluator (engine.py:135-163) — and records:

  * sha256 of the packed scores (f64, row-major) and of the correctness matrix
    (correct_ext as u8), which pin the repo's native window replay
    (paper_2312_05385_b200/synth.py) record for record at full size;
  * the reference compiled kernel's acc/sav (float hex) for all 64 diagonal
    candidates and the 768-row axis family (_exitcore.pyx:27-56), which pin the
    GPU sweep at full size for every candidate.

Uses the reference build of make_golden.py (a copy of /root/reference/pkg under
/tmp, compiled backend asserted). Writes tests/golden/config4_1m.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import load_reference  # noqa: E402


def main(n: int = 1_000_000):
    K = load_reference()
    from conftest import make_chain  # reference test helper
    from eesim.engine import WindowEvaluator
    from eesim.graph import find_feasible_sites
    from eesim.trace import synthesize_workload

    prof = make_chain(13, layer_ms=1.0, ramp_ms=0.01)
    sites = find_feasible_sites(prof)
    curve = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(sites)}
    w = synthesize_workload(prof, n, 0.9, curve, seed=0, miscalibration=0.05, n_labels=10)
    ev = WindowEvaluator(w.records, sites, prof, batch=1)
    cy = K.get_backend("compiled")
    diag = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
    acc, sav = cy.eval_thresholds(ev.scores, ev.correct_ext, ev.serve, ev.vanilla_ms, diag)
    axis = np.full((768, 12), 0.3)
    for j in range(12):
        axis[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
    acc_ax, sav_ax = cy.eval_thresholds(ev.scores, ev.correct_ext, ev.serve, ev.vanilla_ms, axis)
    doc = {
        "n": n, "r": len(sites),
        "scores_sha256": hashlib.sha256(np.ascontiguousarray(ev.scores).tobytes()).hexdigest(),
        "correct_u8_sha256": hashlib.sha256(
            np.ascontiguousarray(ev.correct_ext.astype(np.uint8)).tobytes()).hexdigest(),
        "serve": [float(x).hex() for x in ev.serve], "vanilla": float(ev.vanilla_ms).hex(),
        "diag_acc": [float(x).hex() for x in acc], "diag_sav": [float(x).hex() for x in sav],
        "axis_acc": [float(x).hex() for x in acc_ax], "axis_sav": [float(x).hex() for x in sav_ax],
        "generated_by": "tests/golden/make_config4_golden.py: eesim.trace.synthesize_workload + "
                        "WindowEvaluator + compiled _exitcore.eval_thresholds (reference)",
    }
    with open(os.path.join(HERE, "config4_1m.json"), "w") as fh:
        json.dump(doc, fh, indent=0)
    print("wrote", os.path.join(HERE, "config4_1m.json"))


if __name__ == "__main__":
    main()
