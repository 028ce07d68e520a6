"""One gemm() call per listed shape tag (after warm-up) for ncu captures:
ncu -k regex:k_gemm --launch-skip 2 --launch-count 1 python tools/profile_gemm3.py TAG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_05385_b200.heads import gemm

SHAPES = {"r50_head": (256, 1000, 2048, None), "flush_qkv": (256, 3072, 1024, None),
          "dec_qkv": (32, 3072, 1024, None), "bert_qkv": (8192, 2304, 768, None),
          "bert_fc2": (8192, 768, 3072, None), "bert_fc1": (8192, 3072, 768, "gelu"),
          "lm_head": (32, 50257, 1024, None)}
for tag in sys.argv[1:]:
    m, n, k, act = SHAPES[tag]
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    for _ in range(3):
        gemm(x, w, None, act=act, out_bf16=n % 8 == 0)
    torch.cuda.synchronize()
