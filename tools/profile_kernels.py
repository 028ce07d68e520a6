"""Representative launches of every non-sweep kernel for one ncu capture (not a
benchmark): K4 fused exit controller on a ResNet-50 ramp input (bf16 NCHW
[256, 256, 56, 56] -> 1000 classes would be the GEMM path, so the fused head
here is the 10-class CIFAR-style [256, 512, 4, 4] and a BERT token-0 [64, 768]
-> 2 head), the logits epilogue on a [32, 50257] LM-head ramp, K5 GEMMs (LM head
and a BERT FFN tile), Algorithm 1 on device (1000 x 6), the generic sweep; and
the channels_last ramp paths (NHWC pool of a ResNet-50 [256, 256, 56, 56] map,
fused controller on a ResNet-18 stem map), the K = 1000 logits epilogue, the
axis-family and diagonal sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200.heads import ExitController, exit_from_logits, linear_tc
from paper_2312_05385_b200 import synth
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites

g = torch.Generator(device="cuda").manual_seed(0)
feat = torch.randn(256, 512, 16, device="cuda", generator=g).to(torch.bfloat16).view(256, 512, 4, 4)
ctl = ExitController(torch.randn(10, 512, device="cuda", generator=g) * 0.05)
tok = torch.randn(64, 768, device="cuda", generator=g)
ctl2 = ExitController(torch.randn(2, 768, device="cuda", generator=g) * 0.05, conf="entropy")
lm_x = torch.randn(32, 1024, device="cuda", generator=g).to(torch.bfloat16)
lm_w = (torch.randn(50257, 1024, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
ff_x = torch.randn(8192, 768, device="cuda", generator=g).to(torch.bfloat16)
ff_w = (torch.randn(3072, 768, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
prof = synth.config4_profile(); sites = find_feasible_sites(prof)
arrays = synth.config4_window(1_000_000)
sw = ShardedSweep(arrays, sites, prof)
lat = np.arange(64) / 63.0
th = lat[np.random.default_rng(1).integers(0, 64, size=(64, 12))]
from paper_2312_05385_b200.trace import synthesize_workload
from paper_2312_05385_b200.tuner import TunerParams, tune
from paper_2312_05385_b200.engine import WindowEvaluator
small = synth.config4_window(1000)
ev = WindowEvaluator.from_arrays(small, sites, prof, mode="exact")
from paper_2312_05385_b200.heads import pool_bf16
# channels_last ramp inputs: the ResNet-50 first-bottleneck map through the NHWC pool, and the
# ResNet-18 CIFAR stem map through the fused controller's NHWC path
r50 = torch.randn(256, 256, 56, 56, device="cuda", generator=g).to(torch.bfloat16).contiguous(
    memory_format=torch.channels_last)
r18 = torch.randn(32, 64, 32, 32, device="cuda", generator=g).to(torch.bfloat16).contiguous(
    memory_format=torch.channels_last)
ctl18 = ExitController(torch.randn(10, 64, device="cuda", generator=g) * 0.05)
k1000 = torch.randn(256, 1000, device="cuda", generator=g)
axis = np.full((768, 12), 0.3)
for j in range(12):
    axis[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
diag = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
for it in range(3):
    if it == 2:  # ncu --nvtx --nvtx-include "capture/": one launch of each kernel, warm
        torch.cuda.nvtx.range_push("capture")
    pool_bf16(r50)
    ctl18(r18, 0.5)
    exit_from_logits(k1000, 0.5)
    sw.evaluate_many(axis, to_host=False)
    sw.evaluate_many(diag, to_host=False)
    ctl(feat, 0.5)
    ctl2(tok, 0.5)
    logits = linear_tc(lm_x, lm_w)
    exit_from_logits(logits, 0.5)
    linear_tc(ff_x, ff_w, out_bf16=True)
    tune(None, sites, TunerParams(), prof, evaluator=ev)
    sw.evaluate_many(th, to_host=False)
    if it == 2:
        torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
