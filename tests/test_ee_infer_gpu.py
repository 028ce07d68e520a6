"""End-to-end early-exit inference (BASELINE configs 1-3): the released
(site, label) of every request must equal the reference exit rule
(engine.py:189-220, restated in oracle.exit_record) applied to the
pipeline's own ramp signals; ramp errors must match a torch fp32
restatement of the same heads on the same activations; compaction mode must
release the same results as feedback mode (up to near-threshold rows)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import heads_ref as H
from oracle import oracle as O
from paper_2312_05385_b200 import ee_infer
from paper_2312_05385_b200.graph import ModelProfile, find_feasible_sites

pytestmark = pytest.mark.gpu


def _chain_profile(names):
    nodes = list(names) + ["out"]
    lat = {x: {1: 1.0} for x in nodes}
    ramp = {x: {1: 0.01} for x in nodes[:-1]}
    return ModelProfile(nodes, list(zip(nodes, nodes[1:])), lat, ramp, "out")


def _thresholds(pipe, x, q=(0.05, 0.10, 0.15, 0.20, 0.25, 0.30)):
    probe = pipe.run(x, [0.0] * pipe.n_ramps)
    err = probe.ramp_err.cpu().numpy()
    qs = list(q) + [q[-1]] * max(0, pipe.n_ramps - len(q))
    return [float(np.quantile(err[j], qs[j])) for j in range(pipe.n_ramps)]


def _check_rule(pipe, res, th):
    """Released results == the reference exit rule over the pipeline's signals."""
    prof = _chain_profile(pipe.site_names)
    sites = find_feasible_sites(prof)[: pipe.n_ramps]
    active = list(zip(sites, th))
    recs = res.records(pipe.site_names)
    got_site = res.released_site.cpu().numpy()
    got_label = res.released_label.cpu().numpy()
    for i, rec in enumerate(recs):
        pos, label, _, _ = O.exit_record(rec, active, prof)
        want = pipe.n_ramps if pos is None else pipe.site_names.index(pos)
        assert got_site[i] == want, (i, got_site[i], want)
        assert got_label[i] == label


def test_resnet18_cifar_config1(cuda):
    pipe, model = ee_infer.resnet18_cifar()
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(32, 3, 32, 32, generator=g, device="cuda")
    th = _thresholds(pipe, torch.randn(256, 3, 32, 32, generator=g, device="cuda"))
    res = pipe.run(x, th, timed=True)
    _check_rule(pipe, res, th)
    assert (res.released_site.cpu() >= 0).all() and res.batch_ms > 0
    # ramp errors vs torch fp32 restatement on the same activations
    h = x
    r = 0
    with torch.no_grad():
        for j, stage in enumerate(pipe.stages[:-1]):
            h = stage(h)
            if j in pipe.ramps:
                head = pipe.ramps[j]
                err_ref, _ = H.confidence(H.ramp_head(h, head.weight, head.bias), head.conf)
                assert torch.allclose(res.ramp_err[r].cpu().double(), err_ref, atol=2e-5, rtol=0)
                r += 1
        final = pipe.stages[-1](h).argmax(dim=1).cpu()
    assert torch.equal(res.final_label.cpu().long(), final)
    # compaction mode releases the same results (rows far from a threshold)
    comp = pipe.run(x, th, mode="compact")
    near = np.zeros(32, dtype=bool)
    e = res.ramp_err.cpu().numpy()
    for j, t in enumerate(th):
        near |= np.abs(e[j] - t) < 1e-4
    assert np.array_equal(comp.released_site.cpu().numpy()[~near], res.released_site.cpu().numpy()[~near])
    assert np.array_equal(comp.released_label.cpu().numpy()[~near], res.released_label.cpu().numpy()[~near])


def test_bert_base_config2(cuda):
    pipe, _ = ee_infer.bert_base()
    g = torch.Generator(device="cuda").manual_seed(1)
    ids = torch.randint(0, 30522, (8, 128), generator=g, device="cuda")
    th = _thresholds(pipe, torch.randint(0, 30522, (64, 128), generator=g, device="cuda"))
    res = pipe.run(ids, th)
    _check_rule(pipe, res, th)


def test_resnet50_config3_tensor_core_heads(cuda):
    pipe, _ = ee_infer.resnet50_imagenet()
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(8, 3, 224, 224, generator=g, device="cuda")
    th = _thresholds(pipe, torch.randn(32, 3, 224, 224, generator=g, device="cuda"))
    res = pipe.run(x, th)
    _check_rule(pipe, res, th)


def test_cuda_graph_replay_matches_eager_and_retunes(cuda):
    pipe, _ = ee_infer.resnet18_cifar()
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(32, 3, 32, 32, generator=g, device="cuda")
    th = _thresholds(pipe, torch.randn(256, 3, 32, 32, generator=g, device="cuda"))
    runner = pipe.capture(x, th)
    out = runner.run()
    ref = pipe.run(x, th)
    assert torch.equal(out.released_site, ref.released_site)
    assert torch.equal(out.released_label, ref.released_label)
    assert torch.equal(out.ramp_err, ref.ramp_err)
    # retune without re-capture: thresholds are read from device memory
    th2 = [t * 0.5 for t in th]
    runner.set_thresholds(th2)
    out2 = runner.run()
    ref2 = pipe.run(x, th2)
    assert torch.equal(out2.released_site, ref2.released_site)
    x2 = torch.randn(32, 3, 32, 32, generator=g, device="cuda")
    out3 = runner.run(x2)
    ref3 = pipe.run(x2, th2)
    assert torch.equal(out3.released_label, ref3.released_label)
