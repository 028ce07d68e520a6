"""Swap-AB GEMM at the decode-suffix shapes (M = 160 = 32 x (flush_cap + 1)):
one z tile of 256 rows (path 1) vs five 32-row z tiles (path 6, weights re-read
from L2), in a CUDA graph of 50 calls."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.heads import gemm
out = []
for (m, n, k, act) in [(160, 3072, 1024, None), (160, 1024, 1024, None), (160, 4096, 1024, "gelu_tanh"),
                       (160, 1024, 4096, None), (32, 3072, 1024, None), (64, 3072, 1024, None), (96, 4096, 1024, None)]:
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n, device="cuda")
    row = {"m": m, "n": n, "k": k}
    for path in (1, 6):
        for _ in range(3):
            gemm(a, w, b, act=act, path=path)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50):
                gemm(a, w, b, act=act, path=path)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        row[f"path{path}_us"] = round(e0.elapsed_time(e1) / 50 * 1e3, 2)
    out.append(row)
    print(json.dumps(row))
