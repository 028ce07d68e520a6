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


def _near(fb, th, margin):
    e = fb.ramp_err.float().cpu().numpy()
    near = np.zeros(e.shape[1], dtype=bool)
    for j, t in enumerate(th):
        near |= np.abs(e[j] - t) < margin
    return near


@pytest.mark.parametrize("config", ["resnet18_fp32", "resnet18_bf16", "resnet50_bf16", "bert_bf16"])
def test_compact_runner_matches_feedback_and_censors(cuda, config):
    """CompactRunner (per-(segment, bucket) CUDA graphs, survivors gathered on
    the device) releases what feedback mode releases for every row farther
    than a margin from a threshold (cuDNN/GEMM results may change in the last
    bits with the batch size, hence the margin: 1e-4 fp32, 2e-3 bf16), censors
    later ramps of exited rows (NaN / -1), keeps running under retuned
    thresholds and new inputs, and stops early when every row has exited."""
    g = torch.Generator(device="cuda").manual_seed(11)
    if config.startswith("resnet18"):
        pipe, m = ee_infer.resnet18_cifar()
        b, shape = 32, (3, 32, 32)
    elif config == "resnet50_bf16":
        pipe, m = ee_infer.resnet50_imagenet()
        b, shape = 48, (3, 224, 224)
    else:
        pipe, m = ee_infer.bert_base()
        b = 16
    bf16 = config.endswith("bf16")
    if bf16:
        ee_infer.prepare_bf16(m, channels_last=not config.startswith("bert"))
    margin = 2e-3 if bf16 else 1e-4

    def make(n):
        if config.startswith("bert"):
            return torch.randint(0, 30522, (n, 128), generator=g, device="cuda")
        x = torch.randn(n, *shape, generator=g, device="cuda")
        if bf16:
            x = x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        return x

    th = _thresholds(pipe, make(64))
    x = make(b)
    runner = pipe.capture_compact(x, th)
    for trial, (xx, tt) in enumerate([(x, th), (make(b), th), (x, [t * 0.5 for t in th])]):
        if trial == 2:
            runner.set_thresholds(tt)
        out = runner.run(xx)
        fb = pipe.run(xx, tt)
        near = _near(fb, tt, margin)
        site = out.released_site.cpu().numpy()
        assert (site >= 0).all()
        assert np.array_equal(site[~near], fb.released_site.cpu().numpy()[~near]), trial
        assert np.array_equal(out.released_label.cpu().numpy()[~near],
                              fb.released_label.cpu().numpy()[~near]), trial
        err = out.ramp_err.cpu().numpy()
        for i in range(b):
            s = site[i]
            assert np.isfinite(err[: min(s + 1, pipe.n_ramps), i]).all(), (trial, i)
            assert np.isnan(err[s + 1:, i]).all(), (trial, i)
            assert (out.ramp_label.cpu().numpy()[s + 1:, i] == -1).all()
        fin = out.final_label.cpu().numpy()
        assert ((fin >= 0) == (site == pipe.n_ramps)).all()
        # the eager compaction path agrees as well (same margin)
        ref = pipe.run(xx, tt, mode="compact")
        assert np.array_equal(site[~near], ref.released_site.cpu().numpy()[~near]), trial
    # everything exits at the first ramp: only the first segment runs
    runner.set_thresholds([2.0] * pipe.n_ramps)
    out = runner.run(x)
    assert (out.released_site.cpu() == 0).all()


def test_overlapped_ramps_equal_serial_ramps(cuda):
    """Feedback mode runs the ramp heads on a side stream overlapped with the
    backbone; the results are bit-identical to the serial schedule, eager and
    graph-captured."""
    pipe, m = ee_infer.resnet18_cifar()
    ee_infer.prepare_bf16(m, channels_last=True)
    g = torch.Generator(device="cuda").manual_seed(5)
    mk = lambda n: torch.randn(n, 3, 32, 32, generator=g, device="cuda").to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    th = _thresholds(pipe, mk(128))
    x = mk(32)
    over = pipe.run(x, th, timed=True)
    gr = pipe.capture(x, th).run()
    pipe.overlap_ramps = False
    try:
        ser = pipe.run(x, th)
    finally:
        pipe.overlap_ramps = True
    for a in (over, gr):
        for f in ("released_site", "released_label", "released_err", "ramp_err", "ramp_label", "final_label"):
            assert torch.equal(getattr(a, f), getattr(ser, f)), f
    assert np.all(over.release_ms > 0)


@pytest.mark.parametrize("config", ["resnet18_bf16", "resnet50_bf16", "bert_bf16"])
def test_device_scheduled_compaction_matches_host_schedule(cuda, config):
    """CompactRunner.run_device (one graph: SWITCH nodes pick each segment's
    bucket from the device's live count) releases what the host-scheduled
    runner and feedback mode release off the margin, censors later ramps, and
    skips the remaining segments once every row has exited."""
    g = torch.Generator(device="cuda").manual_seed(5)
    if config == "resnet18_bf16":
        pipe, m = ee_infer.resnet18_cifar()
        b, shape = 32, (3, 32, 32)
    elif config == "resnet50_bf16":
        pipe, m = ee_infer.resnet50_imagenet()
        b, shape = 32, (3, 224, 224)
    else:
        pipe, m = ee_infer.bert_base()
        b = 16
    ee_infer.prepare_bf16(m, channels_last=not config.startswith("bert"))

    def make(n):
        if config.startswith("bert"):
            return torch.randint(0, 30522, (n, 128), generator=g, device="cuda")
        return torch.randn(n, *shape, generator=g, device="cuda").to(torch.bfloat16).contiguous(
            memory_format=torch.channels_last)

    th = _thresholds(pipe, make(64))
    x = make(b)
    runner = pipe.capture_compact(x, th)
    for trial, xx in enumerate([x, make(b), x]):
        dev = runner.run_device(xx)
        site_d = dev.released_site.cpu().numpy().copy()
        err_d = dev.ramp_err.cpu().numpy().copy()
        host = runner.run(xx)
        fb = pipe.run(xx, th)
        near = _near(fb, th, 2e-3)
        assert (site_d >= 0).all()
        assert np.array_equal(site_d[~near], host.released_site.cpu().numpy()[~near]), trial
        assert np.array_equal(site_d[~near], fb.released_site.cpu().numpy()[~near]), trial
        for i in range(b):
            s = site_d[i]
            assert np.isfinite(err_d[: min(s + 1, pipe.n_ramps), i]).all(), (trial, i)
            assert np.isnan(err_d[s + 1:, i]).all(), (trial, i)
    runner.set_thresholds([2.0] * pipe.n_ramps)
    out = runner.run_device(x)
    assert (out.released_site.cpu() == 0).all()
    runner.set_thresholds(th)
    out = runner.run_device(x)
    assert np.array_equal(out.released_site.cpu().numpy()[~_near(pipe.run(x, th), th, 2e-3)],
                          pipe.run(x, th).released_site.cpu().numpy()[~_near(pipe.run(x, th), th, 2e-3)])
