"""GPU parity of the fused ramp head / exit controller (A12-A13) against the
torch fp32 restatement in oracle/heads_ref.py.

Tolerances: logits within 1e-4 relative (fp32 accumulation order differs);
err within 2e-5 absolute; labels and exit masks exact except rows whose
oracle err lies within 1e-5 of the threshold (the north star's near-tie
carve-out, counted and reported); compaction order and scatter exact given
the device's own decisions."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import heads_ref as H
from paper_2312_05385_b200.heads import ExitController, SlotTable, compact_rows, exit_from_logits

pytestmark = pytest.mark.gpu

NEAR = 1e-5


def _check(res, feat, w, bias, conf, thr, alive=None, check_logits=True):
    logits_ref = H.ramp_head(feat, w, bias)
    err_ref, label_ref = H.confidence(logits_ref, conf)
    if check_logits and res.logits is not None:
        got = res.logits.cpu()
        assert torch.allclose(got, logits_ref, rtol=1e-4, atol=1e-4)
    err = res.err.cpu().double()
    assert torch.allclose(err, err_ref, rtol=0, atol=2e-5)
    near = (err_ref - thr).abs() < NEAR
    ex_ref = H.exit_decision(err_ref, thr, alive)
    ex = res.exits.cpu().bool()
    assert torch.equal(ex[~near], ex_ref[~near])
    # labels: exact unless the top-2 logits tie within fp32 noise
    top2 = torch.topk(logits_ref, 2, dim=1).values if logits_ref.shape[1] > 1 else None
    ambiguous = (top2[:, 0] - top2[:, 1]).abs() < 1e-4 if top2 is not None else torch.zeros_like(near)
    assert torch.equal(res.label.cpu().long()[~ambiguous], label_ref[~ambiguous])
    # compaction: stable ascending list of alive rows the device did not exit
    keep_ref = H.compaction(ex, alive)
    assert torch.equal(res.survivors().cpu(), keep_ref)
    return int(near.sum())


HEAD_SHAPES = [(64, 96, 7), (32, 64, 32), (32, 128, 16), (16, 512, 4), (8, 24, 57)]
# pooled rows have no spatial split: one pooled shape
HEAD_CASES = [(lay, sh) for lay in ("nchw", "nhwc") for sh in HEAD_SHAPES] + [("pooled", (64, 96, 7))]


@pytest.mark.parametrize("layout,shape", HEAD_CASES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("conf", ["maxprob", "entropy"])
def test_fused_head_matches_torch(cuda, layout, dtype, conf, shape):
    """Every pooling path, including the cluster-split ones (a row's map split
    over 2 CTAs of one cluster when it is >= 16 KB, up to 8 under
    EEB200_EXIT_MAX_S: the CIFAR ResNet-18 ramp shapes) and a ragged 57x57
    plane."""
    g = torch.Generator().manual_seed(1)
    b, c, hw = shape
    k = 10
    if layout == "pooled":
        feat = torch.randn(b, c, generator=g)
    else:
        feat = torch.randn(b, c, hw, hw, generator=g)
    w = torch.randn(k, c, generator=g) * 0.3
    bias = torch.randn(k, generator=g) * 0.1
    feat_d = feat.to(dtype).cuda()
    if layout == "nhwc":
        feat_d = feat_d.to(memory_format=torch.channels_last)
    head = ExitController(w.cuda(), bias.cuda(), conf=conf, site=3)
    err_probe = head(feat_d, 0.0, want_logits=True).err.cpu()
    thr = float(err_probe.median())
    res = head(feat_d, thr, want_logits=True)
    _check(res, feat_d.float().cpu(), w, bias, conf, thr)


def test_fused_head_wide_clusters_subprocess(cuda):
    """The 4- and 8-CTA cluster splits (EEB200_EXIT_MAX_S=8; the cap is read
    once per process, so in a child pytest)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, EEB200_EXIT_MAX_S="8")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "test_fused_head_matches_torch"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_alive_mask_slots_and_scatter(cuda):
    g = torch.Generator().manual_seed(2)
    b, c, k = 300, 64, 2  # BERT-like binary head, more rows than one CTA scan tile
    feat = torch.randn(b, c, generator=g)
    w = torch.randn(k, c, generator=g)
    head = ExitController(w.cuda(), None, conf="entropy", site=7)
    alive = (torch.rand(b, generator=g) < 0.7).to(torch.uint8).cuda()
    slot = torch.randperm(b, generator=g).to(torch.int32).cuda()
    slots = SlotTable.empty(b)
    probe = head(feat.cuda(), 0.0).err.cpu()
    thr = float(probe.quantile(0.4))
    alive_before = alive.cpu().clone()
    res = head(feat.cuda(), thr, alive=alive, slot=slot, slots=slots)
    _check(res, feat, w, None, "entropy", thr, alive=alive_before)
    ex = res.exits.cpu().bool()
    assert not ex[alive_before == 0].any()  # dead rows never exit again
    # the alive mask is updated in place: exactly the exiting rows were cleared
    assert torch.equal(alive.cpu().bool(), alive_before.bool() & ~ex)
    s = slot.cpu().long()
    site = slots.site.cpu()
    assert (site[s[ex]] == 7).all() and (site[s[~ex]] == -1).all()
    assert torch.equal(slots.label.cpu()[s[ex]], res.label.cpu()[ex])
    assert torch.equal(slots.err.cpu()[s[ex]], res.err.cpu()[ex])


def test_large_head_from_logits_and_row_compaction(cuda):
    g = torch.Generator().manual_seed(3)
    b, k = 256, 1000
    logits = torch.randn(b, k, generator=g) * 3
    probe = exit_from_logits(logits.cuda(), 0.0).err.cpu()
    thr = float(probe.quantile(0.5))
    res = exit_from_logits(logits.cuda(), thr, conf="maxprob")
    err_ref, label_ref = H.confidence(logits, "maxprob")
    assert torch.allclose(res.err.cpu().double(), err_ref, atol=2e-5, rtol=0)
    near = (err_ref - thr).abs() < NEAR
    assert torch.equal(res.exits.cpu().bool()[~near], H.exit_decision(err_ref, thr)[~near])
    # compaction mode: gather the survivors' activations
    act = torch.randn(b, 64, 4, 4, generator=g).cuda()
    dense = compact_rows(act, res.keep, res.n_keep)
    keep = res.survivors().long()
    assert torch.equal(dense[: keep.numel()], act[keep])


def test_exit_rule_is_strict(cuda):
    # a uniform-logit row has err exactly 1 - 1/K; at threshold == err it must not exit
    k = 4
    logits = torch.zeros(2, k).cuda()
    res = exit_from_logits(logits, 1.0 - 1.0 / k, conf="maxprob")
    assert res.exits.cpu().tolist() == [0, 0]
    res = exit_from_logits(logits, np.nextafter(1.0 - 1.0 / k, 2.0), conf="maxprob")
    assert res.exits.cpu().tolist() == [1, 1]


@pytest.mark.parametrize("k,conf", [(50257, "maxprob"), (50257, "entropy"), (3000, "maxprob")])
def test_wide_head_epilogue_matches_torch(cuda, k, conf):
    """The CTA-per-row epilogue for wide heads (LM-head ramps) against torch fp32:
    argmax (first maximum), confidence, strict compare."""
    torch = cuda
    from paper_2312_05385_b200.heads import exit_from_logits

    g = torch.Generator(device="cuda").manual_seed(k)
    logits = torch.randn(32, k, generator=g, device="cuda") * 3.0
    logits[5, 17] = logits[5].max() + 1.0
    logits[5, 18] = logits[5, 17]  # tie: the first index wins
    p = torch.softmax(logits.double(), dim=1)
    if conf == "maxprob":
        err_ref = 1.0 - p.max(dim=1).values
    else:
        err_ref = -(p * torch.log(p.clamp_min(1e-300))).sum(dim=1) / np.log(k)
    thr = float(err_ref.median())
    res = exit_from_logits(logits, thr, conf=conf)
    assert torch.equal(res.label.long().cpu(), torch.argmax(logits, dim=1).cpu())
    assert int(res.label[5]) == 17
    assert torch.allclose(res.err.double().cpu(), err_ref.cpu(), atol=2e-5, rtol=0)
    assert torch.equal(res.exits.bool().cpu(), (res.err.double() < thr).cpu())


@pytest.mark.parametrize("rows,row_elems,seed", [(256, 3136 * 8, 0), (48, 8 * 8 * 256, 1), (7, 64, 2),
                                                 (1000, 16, 3), (32, 16, 4)])
def test_compact_fill_in_place(cuda, rows, row_elems, seed):
    """ee_compact_fill (CompactRunner's in-place compaction) against a host
    restatement: survivors below n_keep stay, the ones above move ascending into
    the exited rows' places below n_keep, request slots follow their rows,
    padding rows read alive = 0 and the dummy slot."""
    from paper_2312_05385_b200.heads import compact_fill

    rng = np.random.default_rng(seed)
    for frac in (0.0, 0.05, 0.5, 0.97, 1.0):
        alive = rng.random(rows) >= frac
        keep = np.flatnonzero(alive).astype(np.int32)
        nk = keep.size
        data = torch.randn(rows, row_elems, device="cuda").to(torch.bfloat16)
        orig = data.clone()
        d_keep = torch.zeros(rows, dtype=torch.int32, device="cuda")
        d_keep[:nk] = torch.from_numpy(keep).cuda()
        d_nk = torch.tensor([nk], dtype=torch.int32, device="cuda")
        rows_in = torch.from_numpy(rng.permutation(rows).astype(np.int32) + 5).cuda()
        rows_out = torch.full((rows,), -7, dtype=torch.int32, device="cuda")
        alive_out = torch.full((rows,), 9, dtype=torch.uint8, device="cuda")
        n_out = torch.zeros(1, dtype=torch.int32, device="cuda")
        compact_fill(data, d_keep, d_nk, rows, rows_in, 12345, rows_out, alive_out, n_out)
        # host restatement of the pairing
        src = np.arange(rows)
        stay = keep[keep < nk]
        holes = np.setdiff1d(np.arange(nk), stay)
        movers = keep[keep >= nk]
        assert holes.size == movers.size
        src[holes] = movers
        ri = rows_in.cpu().numpy()
        want_rows = np.where(np.arange(rows) < nk, ri[src], 12345)
        assert np.array_equal(rows_out.cpu().numpy(), want_rows)
        assert np.array_equal(alive_out.cpu().numpy(), (np.arange(rows) < nk).astype(np.uint8))
        assert int(n_out.item()) == nk
        got = data[:nk].cpu()
        assert torch.equal(got, orig.cpu()[torch.from_numpy(src[:nk]).long()])
