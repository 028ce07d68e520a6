"""Pinned host->device bandwidth for a 96 MB buffer: one copy vs the same bytes
split over 2 / 4 streams (copy engines) vs chunked on one stream."""
import torch, json
n = 96 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); e0.record(); fn(); 
        for s in streams: torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); return n / (ts[len(ts)//2] * 1e-3) / 1e9
def single(): d.copy_(h, non_blocking=True)
def split(k):
    def f():
        cur = torch.cuda.current_stream()
        for i in range(k):
            streams[i].wait_stream(cur)
            with torch.cuda.stream(streams[i]):
                a, b = i * n // k, (i + 1) * n // k
                d[a:b].copy_(h[a:b], non_blocking=True)
    return f
def chunked(k):
    def f():
        for i in range(k):
            a, b = i * n // k, (i + 1) * n // k
            d[a:b].copy_(h[a:b], non_blocking=True)
    return f
print(json.dumps({"single_gbs": t(single), "split2_gbs": t(split(2)), "split4_gbs": t(split(4)),
                  "chunked8_gbs": t(chunked(8))}))
