"""Correctness + timing of the csrc/gemm.cu tcgen05 kernels against cuBLAS
(torch.nn.functional.linear) on the shapes the configs run: BERT-base
projections at B=64 x 128 tokens, GPT-2-medium decode (M = 32) and prefill,
ResNet-50 ramp heads. One JSON line per (shape, path)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2312_05385_b200.heads import gemm


def timeit(fn, iters=20, reps=5):
    """Device time per call: `iters` calls captured in one CUDA graph (no host
    launch overhead), replayed `reps` times, median."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / iters * 1e3)
    return sorted(ts)[len(ts) // 2]


SHAPES = [  # (m, n, k, act, tag)
    (8192, 2304, 768, None, "bert_qkv"), (8192, 768, 768, None, "bert_o"),
    (8192, 3072, 768, "gelu", "bert_fc1"), (8192, 768, 3072, None, "bert_fc2"),
    (32, 3072, 1024, None, "gpt2_dec_qkv"), (32, 1024, 1024, None, "gpt2_dec_o"),
    (32, 4096, 1024, "gelu_tanh", "gpt2_dec_fc1"), (32, 1024, 4096, None, "gpt2_dec_fc2"),
    (32, 50257, 1024, None, "gpt2_lm_head"),
    (4096, 3072, 1024, None, "gpt2_pre_qkv"), (4096, 1024, 4096, None, "gpt2_pre_fc2"),
    (256, 1000, 2048, None, "r50_head"), (256, 3072, 1024, None, "gpt2_flush_qkv"),
    (4096, 4096, 4096, None, "square4k"), (8192, 8192, 8192, None, "square8k"),
]
if __name__ != "__main__":
    SHAPES = []
only = sys.argv[1:]
torch.manual_seed(0)
for m, n, k, act, tag in SHAPES:
    if only and tag not in only:
        continue
    x = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    bias = torch.randn(n, device="cuda") * 0.1
    ref = F.linear(x.float(), w.float(), bias)
    if act == "gelu":
        ref = F.gelu(ref)
    elif act == "gelu_tanh":
        ref = F.gelu(ref, approximate="tanh")
    fl = 2.0 * m * n * k
    wb = bias.to(torch.bfloat16)

    def cub():
        y = F.linear(x, w, wb)
        if act == "gelu":
            y = F.gelu(y)
        elif act == "gelu_tanh":
            y = F.gelu(y, approximate="tanh")
        return y
    t_cub = timeit(cub)
    out_bf16 = n % 8 == 0
    for path in ([0, 1, 2, 4, 3] if m > 256 else [0, 1]):
        if path >= 2 and not out_bf16:
            continue
        try:
            y = gemm(x, w, bias, act=act, out_bf16=out_bf16, path=path)
            torch.cuda.synchronize()
            err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
            t = timeit(lambda: gemm(x, w, bias, act=act, out_bf16=out_bf16, path=path))
            print(json.dumps({"tag": tag, "m": m, "n": n, "k": k, "act": act, "path": path,
                              "max_rel_err": err, "ours_us": round(t, 2),
                              "ours_tflops": round(fl / t / 1e6, 1), "cublas_us": round(t_cub, 2),
                              "cublas_tflops": round(fl / t_cub / 1e6, 1)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"tag": tag, "path": path, "error": str(e)[:300]}), flush=True)
