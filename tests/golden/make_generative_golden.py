"""Golden fixtures for the token-level early-exit timeline (BASELINE config 5),
generated from the REFERENCE itself (pkg/src/eesim/generative.py):

    python tests/golden/make_generative_golden.py

Writes tests/golden/generative.json: token streams (per-token ramp err/label
at every site and the final token), the profile/config/params, and the
reference's run_generative outputs (per-token tpt / exit site / correct, flush
events, critical path). Tests read the JSON only.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402


def main():
    load_reference()
    from conftest import make_chain  # the reference's own test helper
    from eesim.engine import EEConfig
    from eesim.generative import GenParams, run_generative, synthesize_token_trace
    from eesim.graph import find_feasible_sites

    cases = []
    for case_id, (n_layers, ramp_ms, cap, penalty, ramps, ths, seed, k) in enumerate([
        (6, 0.0, 4, {1: 1.0, 4: 1.0}, [2], [0.5], 3, 1),
        (12, 0.2, 2, {1: 1.0, 2: 1.1, 8: 1.6}, [5], [0.4], 11, 1),
        (24, 0.5, 4, {1: 1.0, 5: 1.3}, [11], [0.3], 7, 1),
        (24, 0.5, 3, {1: 1.0, 4: 1.2}, [5, 15], [0.25, 0.35], 19, 1),
        (12, 0.1, 5, {1: 1.0, 6: 1.5}, [3, 8], [0.3, 0.45], 23, 2),
    ]):
        prof = make_chain(n_layers, layer_ms=4.0, ramp_ms=ramp_ms, name="decode")
        sites = find_feasible_sites(prof)
        curve = {s.position: 0.5 + 0.45 * i / max(1, len(sites) - 1) for i, s in enumerate(sites)}
        seqs = synthesize_token_trace(prof, 4, 40, 0.9, curve, seed)
        config = EEConfig(tuple((sites[i], t) for i, t in zip(ramps, ths)))
        params = GenParams(flush_cap=cap, batch_penalty=penalty, score_k=k)
        rep = run_generative(seqs, prof, config, params)
        cases.append({
            "n_layers": n_layers, "ramp_ms": ramp_ms, "flush_cap": cap,
            "penalty": {str(b): m for b, m in penalty.items()}, "ramps": ramps, "thresholds": ths,
            "k": k,
            "sequences": [[{"signals": {p: [s.err, s.label] for p, s in t.ramp_signals.items()},
                            "final": t.final_token} for t in seq] for seq in seqs],
            "tokens": [[t.seq_id, t.index, t.tpt_ms, t.exit_site, t.correct] for t in rep.tokens],
            "flushes": [[e.seq_id, e.site, e.tokens, e.penalty, e.duration_ms, e.kind]
                        for e in rep.flush_events],
            "critical_path_ms": rep.critical_path_ms,
        })
    with open(os.path.join(HERE, "generative.json"), "w") as fh:
        json.dump({"source": "pkg/src/eesim/generative.py run_generative (reference)", "cases": cases},
                  fh, indent=0)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
