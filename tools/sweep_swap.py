"""Split-count sweep of the swap-AB GEMM (graph-timed) for a few small-M shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_05385_b200.heads import gemm
from tools.bench_gemm3 import timeit  # noqa: E402

for m, n, k in [(256, 1000, 2048), (32, 3072, 1024), (32, 1024, 1024), (128, 3072, 1024), (64, 3072, 1024)]:
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    row = {"m": m, "n": n, "k": k}
    for s in [1, 2, 4, 8, 16]:
        try:
            row[f"s{s}"] = round(timeit(lambda: gemm(x, w, None, path=1, splits=s, out_bf16=n % 8 == 0)), 2)
        except Exception as e:  # noqa: BLE001
            row[f"s{s}"] = str(e)[:80]
    print(json.dumps(row), flush=True)
