"""Does the N > 1 sweep step (counts-only sweep -> NCCL all-reduce -> finalise)
capture into a CUDA graph? Run as a 1-rank NCCL group on one GPU (the only
multi-rank shape a 1-GPU box can host): capture K steps, replay, compare with
eager results, time both. One JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import numpy as np, torch
import torch.distributed as dist
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200 import distributed as D
from paper_2312_05385_b200.graph import find_feasible_sites

torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sw = D.ShardedSweep(arrays, sites, prof)
sw._single = lambda: False  # take the multi-rank code path
orig = D.reduce_counts
def forced(hist, ok, group=None):  # the all-reduce even at world size 1
    base = hist.untyped_storage()
    buf = torch.empty(0, dtype=torch.int64, device=hist.device).set_(base, 0, (hist.numel() + ok.numel(),))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return hist, ok
D.reduce_counts = forced
out = {}
ref = sw.evaluate_many(th)
for _ in range(3): sw.evaluate_many(th, to_host=False)
torch.cuda.synchronize()
K = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(K): sw.evaluate_many(th, to_host=False)
b.record(); torch.cuda.synchronize()
out["eager_us_per_step"] = a.elapsed_time(b) / K * 1e3
try:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        res = [sw.evaluate_many(th, to_host=False) for _ in range(K)]
    g.replay(); torch.cuda.synchronize()
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    out["graph_us_per_step"] = a.elapsed_time(b) / K * 1e3
    out["graph_matches_eager"] = all(np.array_equal(x.cpu().numpy(), ref[0]) and np.array_equal(y.cpu().numpy(), ref[1]) for x, y in res)
except Exception as e:  # noqa: BLE001
    out["graph_error"] = f"{type(e).__name__}: {e}"[:300]
# the same with the exchange on a side stream (overlap_comm): sweep k+1 runs
# while sweep k is all-reduced and finalised
sw2 = D.ShardedSweep(arrays, sites, prof, overlap_comm=True)
sw2._single = lambda: False
assert all(np.array_equal(a, b) for a, b in zip(sw2.evaluate_many(th), ref))
for _ in range(3): sw2.evaluate_many(th, to_host=False)
sw2.join(); torch.cuda.synchronize()
try:
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        res2 = [sw2.evaluate_many(th, to_host=False) for _ in range(K)]
        sw2.join()
    g2.replay(); torch.cuda.synchronize()
    a.record(); g2.replay(); b.record(); torch.cuda.synchronize()
    out["overlap_graph_us_per_step"] = a.elapsed_time(b) / K * 1e3
    out["overlap_graph_matches_eager"] = all(np.array_equal(x.cpu().numpy(), ref[0]) and np.array_equal(y.cpu().numpy(), ref[1]) for x, y in res2)
except Exception as e:  # noqa: BLE001
    out["overlap_graph_error"] = f"{type(e).__name__}: {e}"[:300]
print(json.dumps(out))
dist.destroy_process_group()
