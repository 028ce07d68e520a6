"""Per-call cost of the fused exit controller on the six ResNet-18 CIFAR ramp
inputs (bf16 channels_last, batch 32, 10 classes), captured in a CUDA graph of
200 calls: the ramp overhead a feedback-mode batch pays per site."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.heads import ExitController, SlotTable

g = torch.Generator(device="cuda").manual_seed(0)
shapes = [(64, 32, 32), (64, 32, 32), (128, 16, 16), (256, 8, 8), (256, 8, 8), (512, 4, 4)]
out = {}
for c, h, w in shapes:
    x = torch.randn(32, c, h, w, generator=g, device="cuda").to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    ctl = ExitController(torch.randn(10, c, generator=g, device="cuda") * 0.05)
    th = torch.tensor([0.05], dtype=torch.float64, device="cuda")
    alive = torch.ones(32, dtype=torch.uint8, device="cuda")
    rows = torch.arange(32, dtype=torch.int32, device="cuda")
    slots = SlotTable.empty(32)
    err = torch.empty(32, dtype=torch.float32, device="cuda")
    lab = torch.empty(32, dtype=torch.int32, device="cuda")
    for compact in (True, False):
        kw = dict(alive=alive, slot=rows, slots=slots, compact=compact)
        if not compact:
            kw.update(out_err=err, out_label=lab)
        for _ in range(3):
            ctl(x, th, **kw)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(200):
                ctl(x, th, **kw)
        gr.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        out[f"{c}x{h}x{w}" + ("" if compact else "_feedback")] = round(a.elapsed_time(b) / 200 * 1e3, 2)
print(json.dumps({"us_per_ramp_call": out}))
