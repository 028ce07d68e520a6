"""Per-kernel time of the EE ramps in one feedback-mode batch (configs 1 and 3,
bf16 channels_last backbones), from the library's own profiling events."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200 import ee_infer, _native as nat

torch.backends.cudnn.benchmark = True
g = torch.Generator(device="cuda").manual_seed(0)
for name, build, shape, b in (("resnet18", ee_infer.resnet18_cifar, (3, 32, 32), 32),
                              ("resnet50", ee_infer.resnet50_imagenet, (3, 224, 224), 256)):
    pipe, m = build()
    m.to(memory_format=torch.channels_last).to(torch.bfloat16)
    x = torch.randn(b, *shape, generator=g, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    th = [0.0] * pipe.n_ramps
    for _ in range(3): pipe.run(x, th)
    torch.cuda.synchronize()
    nat.profile_read(); nat.profile_enable(True)
    for _ in range(5): pipe.run(x, th)
    torch.cuda.synchronize()
    nat.profile_enable(False)
    k = nat.profile_read()
    print(name, json.dumps({a: {"launches": v["launches"] // 5, "us_per_batch": round(1e3 * v["ms"] / 5, 1)} for a, v in k.items()}))
