"""Time the tcgen05 ramp-head GEMM (ours) against torch.matmul (cuBLAS) on the
same bf16 operands; prints one JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_05385_b200.heads import linear_tc


def timeit(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


for m, n, k in [(256, 1000, 2048), (256, 1000, 1024), (32, 10, 512), (4096, 4096, 4096), (8192, 8192, 8192)]:
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    ours = timeit(lambda: linear_tc(x, w))
    cub = timeit(lambda: torch.matmul(x, w.t()).float())
    fl = 2.0 * m * n * k
    print(json.dumps({"m": m, "n": n, "k": k, "ours_us": ours * 1e3, "ours_tflops": fl / ours / 1e9,
                      "cublas_us": cub * 1e3, "cublas_tflops": fl / cub / 1e9}))
