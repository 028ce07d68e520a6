"""torch fp32 CPU restatement of a ramp head + exit decision — TEST
INFRASTRUCTURE ONLY (the parity checker for paper_2312_05385_b200.heads).

There is no reference code for ramp heads (SPEC.md:9 abstracts ramps to
(err, label) signals); the paper defines them as a final FC prepended with a
lightweight pooling with max-probability or entropy confidence
(PAPER.md:331). The exit rule and the released fields follow
pkg/src/eesim/engine.py:189-220: exit iff err < threshold (strict).
"""

from __future__ import annotations

import math

import torch


def ramp_head(feat, weight, bias=None):
    """Global average pool over H, W (if 4-D) then FC, in fp32 on the CPU."""
    x = feat.detach().float().cpu()
    if x.dim() == 4:
        x = x.mean(dim=(2, 3))
    w = weight.detach().float().cpu()
    out = x @ w.t()
    if bias is not None:
        out = out + bias.detach().float().cpu()
    return out


def confidence(logits, conf="maxprob"):
    """(err, label): err = 1 - max softmax, or entropy / ln K; label = argmax."""
    l = logits.double()
    p = torch.softmax(l, dim=1)
    label = torch.argmax(l, dim=1)
    if conf == "maxprob":
        err = 1.0 - p.max(dim=1).values
    else:
        k = l.shape[1]
        h = -(p * torch.log(p.clamp_min(1e-300))).sum(dim=1)
        err = h / math.log(k) if k > 1 else torch.zeros_like(h)
    return err.clamp(0.0, 1.0), label


def exit_decision(err, threshold, alive=None):
    ex = err < threshold
    if alive is not None:
        ex &= alive.bool().cpu()
    return ex


def compaction(exits, alive=None):
    keep = ~exits
    if alive is not None:
        keep &= alive.bool().cpu()
    return torch.nonzero(keep).flatten().to(torch.int32)
