"""Where a compaction-mode batch spends its time: per segment, the bucket the
CompactRunner ran it at, the live rows after it, and its CUDA-event time, next
to the feedback graph's and the vanilla graph's batch time.
Usage: profile_compact.py [1|2|3]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2312_05385_b200 import ee_infer

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_ee import _image, quantile_thresholds  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "3"
g = torch.Generator(device="cuda").manual_seed(0)
img = _image(g, True)
if which == "3":
    pipe, m = ee_infer.resnet50_imagenet(); ee_infer.prepare_bf16(m, True)
    make, B = (lambda b: img(b, (3, 224, 224))), 256
elif which == "1":
    pipe, m = ee_infer.resnet18_cifar(); ee_infer.prepare_bf16(m, True)
    make, B = (lambda b: img(b, (3, 32, 32))), 32
else:
    pipe, m = ee_infer.bert_base(); ee_infer.prepare_bf16(m, False)
    make, B = (lambda b: torch.randint(0, 30522, (b, 128), generator=g, device="cuda")), 64
th = quantile_thresholds(pipe, make(max(B, 64)))
x = make(B)
crun = pipe.capture_compact(x, th)
for _ in range(5):
    crun.run()
torch.cuda.synchronize()
# one instrumented run: the same loop as CompactRunner.run with events per segment
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(crun.segments) + 1)]
crun.graphs["reset"].replay()
evs[0].record()
bb, used = crun.B, []
for k in range(len(crun.segments)):
    if k >= 2:
        crun.done[k - 2].synchronize()
        n = int(crun.n_host[k - 2])
        if n == 0:
            break
        bb = crun.bucket(n)
    crun._graph(k, bb).replay()
    crun.done[k].record()
    evs[k + 1].record()
    used.append(bb)
torch.cuda.synchronize()
live = crun.n_live.cpu().tolist()
seg = []
for k, bb in enumerate(used):
    seg.append({"segment": crun.segments[k], "bucket": bb, "live_after": live[k] if k < len(live) else None,
                "ms": round(evs[k].elapsed_time(evs[k + 1]), 4)})
site = crun.out.released_site.cpu().numpy()
print(json.dumps({"config": which, "batch": B, "total_ms": round(evs[0].elapsed_time(evs[len(used)]), 4),
                  "released_per_site": np.bincount(site, minlength=pipe.n_ramps + 1).tolist(),
                  "segments": seg}))
