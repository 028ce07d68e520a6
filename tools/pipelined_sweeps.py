"""Back-to-back config-4 sweeps: eager vs CUDA graph, resident overlap on/off,
1..8 rotated window copies; checks every replayed result against one eager sweep."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, engine, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites

prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sweeps = [ShardedSweep(arrays, sites, prof) for _ in range(8)]
if "DIAG_VERSION" in os.environ:
    nat.set_diag_version(int(os.environ["DIAG_VERSION"]))
engine.RESIDENT_OVERLAP = False
ref_acc, ref_sav = sweeps[0].evaluate_many(th)
K = int(os.environ.get("K", "300"))
out = {}
for overlap in (False, True):
    engine.RESIDENT_OVERLAP = overlap
    for copies in [int(x) for x in os.environ.get("COPIES", "1,2,4,8").split(",")]:
        for mode in os.environ.get("MODES", "eager,graph").split(","):
            def run():
                return [sweeps[i % copies].evaluate_many(th, to_host=False) for i in range(K)]
            for _ in range(3): run()
            torch.cuda.synchronize()
            if mode == "graph":
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    res = run()
                g.replay(); torch.cuda.synchronize()
                fn = g.replay
            else:
                res = None
                fn = run
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(3):
                torch.cuda.synchronize(); a.record(); r = fn(); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) / K * 1e3)
                if res is None: res = r
            ok = all(np.array_equal(x.cpu().numpy(), ref_acc) and np.array_equal(y.cpu().numpy(), ref_sav)
                     for x, y in res)
            key = f"overlap={int(overlap)} copies={copies} {mode}"
            out[key] = {"us_per_sweep": round(min(ts), 2), "all_equal": ok}
            print(key, out[key], flush=True)
            del res
print(json.dumps(out))
