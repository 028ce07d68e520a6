"""One feedback-mode ResNet-18 batch replayed as a CUDA graph (for an ncu
launch list of every node: which kernels the ramps add to the backbone)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200 import ee_infer

torch.backends.cudnn.benchmark = True
g = torch.Generator(device="cuda").manual_seed(0)
pipe, m = ee_infer.resnet18_cifar()
m.to(memory_format=torch.channels_last).to(torch.bfloat16)
x = torch.randn(32, 3, 32, 32, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
runner = pipe.capture(x, [0.05] * pipe.n_ramps)
for _ in range(3):
    runner.run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("replay")
runner.run()
torch.cuda.synchronize()
print("done")
