"""One vanilla and one feedback-mode batch of a config, each replayed as a CUDA
graph (for an ncu launch list of every node: where the backbone's time goes
and which kernels the ramps add). Usage: profile_ee_graph.py [1|2|3]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200 import ee_infer

torch.backends.cudnn.benchmark = True
which = sys.argv[1] if len(sys.argv) > 1 else "1"
g = torch.Generator(device="cuda").manual_seed(0)
if which == "1":
    pipe, m = ee_infer.resnet18_cifar()
    ee_infer.prepare_bf16(m, True)
    x = torch.randn(32, 3, 32, 32, generator=g, device="cuda")
elif which == "3":
    pipe, m = ee_infer.resnet50_imagenet()
    ee_infer.prepare_bf16(m, True)
    x = torch.randn(256, 3, 224, 224, generator=g, device="cuda")
else:
    pipe, m = ee_infer.bert_base()
    ee_infer.prepare_bf16(m, False)
    x = torch.randint(0, 30522, (64, 128), generator=g, device="cuda")
if x.is_floating_point():
    x = x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
runner = pipe.capture(x, [0.05] * pipe.n_ramps)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.no_grad(), torch.cuda.stream(s):
    for _ in range(2):
        h = x
        for st in pipe.stages:
            h = st(h)
torch.cuda.current_stream().wait_stream(s)
vg = torch.cuda.CUDAGraph()
with torch.no_grad(), torch.cuda.graph(vg):
    h = x
    for st in pipe.stages:
        h = st(h)
for _ in range(3):
    runner.run()
    vg.replay()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("vanilla")
vg.replay()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("ee")
runner.run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
