"""N = 64 GEMMs (ResNet-50 layer1 1x1 256 -> 64 at B=256, the stem's K = 168): the
planner's 256x64 tile against 256x128 / 256x256 tiles whose extra columns are
TMA zero-fill, warm, CUDA-graph timed (is the 64-wide MMA itself the limit?)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.heads import gemm


def timeit(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
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


for tag, m, n, k in (("l1_conv1", 802816, 64, 256), ("stem", 3211264, 64, 168), ("n128", 802816, 128, 256)):
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    b = torch.randn(n, device="cuda")
    ref = gemm(x, w, b, act="relu", path=0)
    out = {"tag": tag, "m": m, "n": n, "k": k}
    for name, path in (("auto", 0), ("bn256", 2), ("bn128", 3), ("bn64", 5)):
        y = gemm(x, w, b, act="relu", path=path)
        out[name + "_us"] = round(timeit(lambda: gemm(x, w, b, act="relu", path=path)), 2)
        out[name + "_same"] = bool(torch.equal(y, ref))
    out["bytes_mb"] = round((m * k + m * n) * 2 / 1e6, 1)
    print(json.dumps(out))

# the 64-wide 3x3 implicit GEMM (layer1, B=256, 56x56) warm, against cuDNN on the same operands
from paper_2312_05385_b200 import convnet

CL = torch.channels_last
for cin, cout, hw in ((64, 64, 56), (128, 128, 28), (256, 256, 14)):
    conv = torch.nn.Conv2d(cin, cout, 3, 1, 1).cuda().to(torch.bfloat16).to(memory_format=CL)
    x = torch.randn(256, cin, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=CL)
    c = convnet.Conv(conv)
    ours = timeit(lambda: c(x, act="relu"))
    lib = timeit(lambda: torch.relu(conv(x)))
    fl = 2 * 256 * hw * hw * cout * cin * 9
    print(json.dumps({"tag": f"conv3x3_{cin}_{hw}", "ours_us": round(ours, 2), "cudnn_relu_us": round(lib, 2),
                      "ours_tflops": round(fl / ours / 1e6, 1)}))
