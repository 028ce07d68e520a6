"""Phase timeline of back-to-back resident sweeps (EE_MODE_FLAG_RESIDENT), each
launch with its own %globaltimer trace buffer, relative to the first launch."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, engine, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites
prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sw = ShardedSweep(arrays, sites, prof)
engine.RESIDENT_OVERLAP = os.environ.get("OVERLAP", "1") == "1"
lib = nat.load_library()
L = 8
trs = [torch.zeros(160 * 6, dtype=torch.int64, device="cuda") for _ in range(L)]
for _ in range(5): sw.evaluate_many(th, to_host=False)
torch.cuda.synchronize()
for i in range(L):
    nat.check(lib.ee_diag_trace(nat.workspace(), trs[i].data_ptr()))
    sw.evaluate_many(th, to_host=False)
nat.check(lib.ee_diag_trace(nat.workspace(), None))
torch.cuda.synchronize()
ts = [t.cpu().numpy().reshape(160, 6).astype(np.float64) for t in trs]
t0 = min(t[t[:, 0] > 0, 0].min() for t in ts)
rows = []
for i, t in enumerate(ts):
    t = t[t[:, 0] > 0]
    g = (t - t0) / 1e3
    last = int(np.argmax(g[:, 4]))
    rows.append({"launch": i, "ctas": len(t), "start_min": g[:, 0].min(), "start_med": float(np.median(g[:, 0])),
                 "start_max": g[:, 0].max(), "prologue_end_med": float(np.median(np.delete(g[:, 1], last))),
                 "loop_end_med": float(np.median(g[:, 2])), "loop_end_max": g[:, 2].max(),
                 "merged_med": float(np.median(g[:, 3])), "merged_max": g[:, 3].max(),
                 "last_cta_waited": g[last, 1], "final_end": g[last, 4]})
for r in rows:
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))
