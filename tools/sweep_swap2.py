"""Swap-AB GEMM latency anatomy: time vs K (k-tiles per CTA) at S=1 and vs M."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_05385_b200.heads import gemm
from tools.bench_gemm3 import timeit  # noqa: E402

for m in (32, 128):
    for n in (1024, 3072):
        row = {"m": m, "n": n}
        for k in (64, 256, 1024, 4096):
            x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
            row[f"k{k}"] = round(timeit(lambda: gemm(x, w, None, path=1, splits=1)), 2)
        print(json.dumps(row), flush=True)
