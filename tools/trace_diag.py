"""Phase timeline of the diagonal sweep kernels from per-CTA %globaltimer
stamps (ee_diag_trace): us from the first CTA's start. Slots per CTA: 0 start,
1 prologue done (the finalising CTA: its turn to finalise), 2 last warp out of
the loop, 3 folded, 4 finalised (finalising CTA), 5 merged + fenced (k_diag3
version 6)."""
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
tr = torch.zeros(160 * 6, dtype=torch.int64, device="cuda")
for ver in [int(v) for v in (sys.argv[1:] or ["4", "6"])]:
    nat.set_diag_version(ver)
    for _ in range(5): sw.evaluate_many(th, to_host=False)
    res = []
    for it in range(5):
        nat.l2_flush(flush); tr.zero_(); torch.cuda.synchronize()
        nat.check(nat.load_library().ee_diag_trace(nat.workspace(), tr.data_ptr()))
        sw.evaluate_many(th, to_host=False); torch.cuda.synchronize()
        nat.check(nat.load_library().ee_diag_trace(nat.workspace(), None))
        t = tr.cpu().numpy().reshape(160, 6).astype(np.float64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
        last = int(np.nanargmax(t[:, 4]))
        res.append({"ctas": len(t), "start_spread": np.nanmax(t[:, 0]),
                    "prologue_end_med": float(np.nanmedian(np.delete(t[:, 1], last))),
                    "loop_end_med": float(np.nanmedian(t[:, 2])), "loop_end_max": np.nanmax(t[:, 2]),
                    "folded_med": float(np.nanmedian(t[:, 3])), "folded_max": np.nanmax(t[:, 3]),
                    "merged_med": float(np.nanmedian(t[:, 5])) if ver == 6 else None,
                    "merged_max": np.nanmax(t[:, 5]) if ver == 6 else None,
                    "last_cta_turn": t[last, 1], "last_loop_end": t[last, 2], "final_end": t[last, 4]})
    print(json.dumps({"version": ver, "runs": [{k: (round(float(v), 2) if v is not None else None)
                                                 for k, v in r.items()} for r in res[-3:]]}))
