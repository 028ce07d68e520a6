"""tcgen05 GEMM (ours, linear_tc) vs cuBLAS on the decode / encoder shapes the
backbones use (GPT-2-medium decode at batch 32 and 160, BERT-base at 64 x 128)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.heads import linear_tc


def timeit(fn, iters=int(os.environ.get("ITERS", 100))):
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


for m, n, k in [(32, 3072, 1024), (32, 1024, 1024), (32, 4096, 1024), (32, 1024, 4096), (32, 50257, 1024),
                (160, 4096, 1024), (8192, 2304, 768), (8192, 768, 768), (8192, 3072, 768), (8192, 768, 3072)]:
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    ours = timeit(lambda: linear_tc(x, w))
    cub = timeit(lambda: torch.nn.functional.linear(x, w))
    byt = 2 * (m * k + n * k) + 4 * m * n
    print(json.dumps({"m": m, "n": n, "k": k, "ours_us": round(ours * 1e3, 2), "cublas_bf16out_us": round(cub * 1e3, 2),
                      "ours_GBps": round(byt / ours / 1e6), "ours_tflops": round(2 * m * n * k / ours / 1e9, 1)}))
