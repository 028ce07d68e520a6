"""Config-4 sweeps of K windows in one persistent launch (ee_eval_thresholds_windows)
over 4 rotated resident copies of the 1M x 12 window, against K sweeps captured
in one CUDA graph (what bench.py times); both checked against one sweep."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, kernels as K
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites

prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
evs = [WindowEvaluator.from_arrays(arrays, sites, prof, mode="hist") for _ in range(4)]
ref_acc, ref_sav = evs[0].evaluate_many(th)
out = {}
for k in (100, 500):
    order = [i % 4 for i in range(k)]
    for _ in range(2):
        acc, sav = K.eval_thresholds_windows(evs, th, order)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        a.record(); acc, sav = K.eval_thresholds_windows(evs, th, order); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / k * 1e3)
    ok = bool((acc.cpu().numpy() == ref_acc[None, :]).all() and (sav.cpu().numpy() == ref_sav[None, :]).all())
    out[f"K{k}"] = {"us_per_window": round(min(ts), 2), "candidates_per_s": 64 / (min(ts) * 1e-6),
                    "identical_to_single_sweep": ok}
print(json.dumps(out))
