"""Warm (L2-resident, graph of 20 calls) and cold (256 MiB L2 flush before each
call) device time of the BERT add+LayerNorm (8192 x 768) and the ResNet-50
classifier pool (256 x 2048 x 7 x 7, channels_last) against torch's kernels."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.heads import pool_bf16

lib = nat.load_library()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def warm(fn, iters=20):
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000 / iters)
    return sorted(ts)[2]


def cold(fn, reps=11):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    return sorted(ts)[reps // 2]


rows, d = 8192, 768
h = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
y = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
gm = torch.ones(d, device="cuda").to(torch.bfloat16)
bt = torch.zeros(d, device="cuda").to(torch.bfloat16)
x = torch.empty_like(h)
st = nat.stream_handle(torch)
ln = lambda: lib.ee_add_layernorm_bf16(h.data_ptr(), y.data_ptr(), gm.data_ptr(), bt.data_ptr(), 1e-12, rows, d,
                                       x.data_ptr(), nat.stream_handle(torch))
tln = lambda: torch.nn.functional.layer_norm(h + y, (d,), gm, bt, 1e-12)
fm = torch.randn(256, 2048, 7, 7, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
pl = lambda: pool_bf16(fm)
tpl = lambda: fm.mean((2, 3))
shapes = {"pool_256x1024x14x14": (256, 1024, 14), "pool_256x512x28x28": (256, 512, 28)}
extra = {}
for tag, (b_, c_, s_) in shapes.items():
    m_ = torch.randn(b_, c_, s_, s_, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    f1, f2 = (lambda m_=m_: pool_bf16(m_)), (lambda m_=m_: m_.mean((2, 3)))
    extra[tag] = {"bytes": m_.numel() * 2, "ours_warm_us": warm(f1), "ours_cold_us": cold(f1),
                  "torch_warm_us": warm(f2), "torch_cold_us": cold(f2)}
out = {"add_layernorm_8192x768": {"bytes": 4 * rows * d * 2, "ours_warm_us": warm(ln), "ours_cold_us": cold(ln),
                                   "torch_warm_us": warm(tln), "torch_cold_us": cold(tln)},
       "pool_256x2048x7x7": {"bytes": fm.numel() * 2, "ours_warm_us": warm(pl), "ours_cold_us": cold(pl),
                             "torch_warm_us": warm(tpl), "torch_cold_us": cold(tpl)}}
out.update(extra)
for k, v in out.items():
    v["ours_cold_gbs"] = v["bytes"] / v["ours_cold_us"] / 1e3
print(json.dumps(out))
