"""Closed-loop serving (serve_live.py): every exit the GPU exit controllers
take matches the reference exit rule (engine.py:189-220, oracle.exit_record)
under the thresholds that batch ran with, and every retune the monitor
triggers equals Algorithm 1 (oracle.tune, pinned to the reference) on the
same history; the next batch runs with the retuned thresholds."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("graphs", [False, True], ids=["eager", "graphs"])
def test_closed_loop_decisions_and_retunes_match_reference(cuda, graphs):
    torch = cuda
    from paper_2312_05385_b200 import ee_infer
    from paper_2312_05385_b200.serve_live import LiveParams, profile_pipeline, serve_live
    from paper_2312_05385_b200.tuner import TunerParams

    pipe, _ = ee_infer.resnet18_cifar()
    g = torch.Generator(device="cuda").manual_seed(3)
    n = 320
    x = torch.randn(n, 3, 32, 32, generator=g, device="cuda")
    prof = profile_pipeline(pipe, x[:32])
    probe = pipe.run(x[:64], [0.0] * pipe.n_ramps)
    err = probe.ramp_err.float().cpu().numpy()
    th0 = [float(np.quantile(err[j], 0.3)) for j in range(pipe.n_ramps)]
    arrivals = np.cumsum(np.random.default_rng(4).exponential(0.05, size=n))
    params = LiveParams(max_batch=32, acc_constraint=0.97,
                        tuner=TunerParams(acc_loss_budget=0.05, accuracy_window=16, tuning_history=96))
    rep = serve_live(pipe, x, arrivals, prof, th0, params, graphs=graphs)
    assert len(rep.rows) == n
    assert all(b.busy_ms > 0 for b in rep.batches)
    sites = [s for s in __import__("paper_2312_05385_b200.graph", fromlist=["x"]).find_feasible_sites(prof)
             if s.position in {f"st{j}" for j in pipe.ramp_order}]
    R = len(sites)
    for b in rep.batches:
        active = list(zip(sites, b.thresholds))
        for rec, site in zip(b.records, b.released_site):
            pos, _, _, _ = O.exit_record(rec, active, prof, 1, 1)
            want = R if pos is None else [s.position for s in sites].index(pos)
            assert int(site) == want
    assert rep.tunes, "the monitor never triggered a retune"
    for t in rep.tunes:
        th, sav, acc, *_ = O.tune(t["history"], sites, prof, budget=0.05, init_step=0.1,
                                  min_step=0.01)
        assert th == t["thresholds"]
    # a retune takes effect from the next batch on: every batch runs with the
    # thresholds of the last retune before its first request
    for b in rep.batches:
        prior = [t for t in rep.tunes if t["after_request"] < b.records[0].id]
        if prior:
            assert b.thresholds == tuple(prior[-1]["thresholds"])
    starts = [b.start_ms for b in rep.batches]
    assert starts == sorted(starts)
