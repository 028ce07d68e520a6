"""Representative launches of every non-sweep kernel for one ncu capture (not a
benchmark): K4 fused exit controller on a ResNet-50 ramp input (bf16 NCHW
[256, 256, 56, 56] -> 1000 classes would be the GEMM path, so the fused head
here is the 10-class CIFAR-style [256, 512, 4, 4] and a BERT token-0 [64, 768]
-> 2 head), the logits epilogue on a [32, 50257] LM-head ramp, K5 GEMMs (LM head
and a BERT FFN tile), Algorithm 1 on device (1000 x 6), the generic sweep."""
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
for _ in range(3):
    ctl(feat, 0.5)
    ctl2(tok, 0.5)
    logits = linear_tc(lm_x, lm_w)
    exit_from_logits(logits, 0.5)
    linear_tc(ff_x, ff_w, out_bf16=True)
    tune(None, sites, TunerParams(), prof, evaluator=ev)
    sw.evaluate_many(th, to_host=False)
torch.cuda.synchronize()
print("done")
