"""The token-level timeline oracle (oracle/generative_ref.py) against the
reference's own run_generative outputs (tests/golden/generative.json, made by
tests/golden/make_generative_golden.py from pkg/src/eesim/generative.py).
CPU only: this pins the checker the GPU decoder tests use."""

from __future__ import annotations

import json
import os
from types import SimpleNamespace

import pytest

from conftest import GOLDEN, make_chain
from oracle.generative_ref import sequence_timeline
from paper_2312_05385_b200.engine import EEConfig
from paper_2312_05385_b200.graph import find_feasible_sites, interp_ms
from paper_2312_05385_b200.trace import RampSignal


def _cases():
    with open(os.path.join(GOLDEN, "generative.json")) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", range(5))
def test_timeline_oracle_matches_reference(case):
    c = _cases()[case]
    prof = make_chain(c["n_layers"], layer_ms=4.0, ramp_ms=c["ramp_ms"], name="decode")
    sites = find_feasible_sites(prof)
    config = EEConfig(tuple((sites[i], t) for i, t in zip(c["ramps"], c["thresholds"])))
    pairs = tuple(sorted((int(b), float(m)) for b, m in c["penalty"].items()))
    toks, flushes, clock = [], [], 0.0
    for sid, seq in enumerate(c["sequences"]):
        tokens = [SimpleNamespace(ramp_signals={p: RampSignal(e, l) for p, (e, l) in t["signals"].items()},
                                  final_token=t["final"]) for t in seq]
        st, fl, ck = sequence_timeline(tokens, prof, config, flush_cap=c["flush_cap"],
                                       penalty=lambda b: interp_ms(pairs, b), k=c["k"])
        toks += [[sid, s.index, s.tpt_ms, s.exit_site, s.correct] for s in st]
        flushes += [[sid, f.site, f.tokens, f.penalty, f.duration_ms, f.kind] for f in fl]
        clock += ck
    assert toks == c["tokens"]
    assert flushes == c["flushes"]
    assert clock == c["critical_path_ms"]
