"""Phase timeline of k_diag2 from per-CTA %globaltimer stamps (ee_diag_trace)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites
prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sw = ShardedSweep(arrays, sites, prof)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tr = torch.zeros(148 * 6, dtype=torch.int64, device="cuda")
for ver in [int(v) for v in (sys.argv[1:] or ["2", "3"])]:
    nat.set_diag_version(ver)
    for _ in range(5): sw.evaluate_many(th, to_host=False)
    res = []
    for it in range(5):
        flush.zero_(); tr.zero_(); torch.cuda.synchronize()
        nat.check(nat.load_library().ee_diag_trace(nat.workspace(), tr.data_ptr()))
        sw.evaluate_many(th, to_host=False); torch.cuda.synchronize()
        nat.check(nat.load_library().ee_diag_trace(nat.workspace(), None))
        t = tr.cpu().numpy().reshape(148, 6).astype(np.float64)
        t0 = t[:, 0].min()
        t = (t - t0) / 1e3  # us
        last = int(np.argmax(t[:, 4]))
        res.append({"start_spread": t[:, 0].max(), "prologue_end_med": float(np.median(np.delete(t[:, 1], last))),
                    "loop_end_med": float(np.median(t[:, 2])), "loop_end_max": t[:, 2].max(),
                    "merged_med": float(np.median(t[:, 3])), "merged_max": t[:, 3].max(),
                    "last_cta_fenced": t[last, 1], "last_cta_scanned": t[last, 5], "last_loop_end": t[last, 2],
                    "last_merged": t[last, 3], "final_end": t[last, 4]})
    print(json.dumps({"version": ver, "runs": [{k: round(v, 2) for k, v in r.items()} for r in res[-2:]]}))
