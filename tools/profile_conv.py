"""One routed 3x3 convolution (implicit GEMM over TMA im2col loads) and one
1x1 + shortcut GEMM at ResNet-50 layer1 shapes, B=256, for an ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200 import convnet

CL = torch.channels_last
g = torch.Generator(device="cuda").manual_seed(0)
which = sys.argv[1] if len(sys.argv) > 1 else "3x3"
if which == "3x3":
    conv = torch.nn.Conv2d(64, 64, 3, 1, 1).cuda().to(torch.bfloat16).to(memory_format=CL)
    x = torch.randn(256, 64, 56, 56, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=CL)
    c = convnet.Conv(conv)
    for _ in range(3):
        y = c(x, act="relu")
elif which == "1x1_64":  # layer1 bottleneck conv1: 256 -> 64 channels (a 64-wide tile)
    conv = torch.nn.Conv2d(256, 64, 1).cuda().to(torch.bfloat16).to(memory_format=CL)
    x = torch.randn(256, 256, 56, 56, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=CL)
    c = convnet.Conv(conv)
    for _ in range(3):
        y = c(x, act="relu")
else:
    conv = torch.nn.Conv2d(64, 256, 1).cuda().to(torch.bfloat16).to(memory_format=CL)
    x = torch.randn(256, 64, 56, 56, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=CL)
    r = torch.randn(256, 256, 56, 56, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=CL)
    c = convnet.Conv(conv)
    for _ in range(3):
        y = c(x, act="relu", res=r)
torch.cuda.synchronize()
print("done", which)
