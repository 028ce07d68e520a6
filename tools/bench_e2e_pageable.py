"""The drop-in call with ordinary (pageable) numpy buffers vs pinned ones:
kernels.eval_thresholds on the config-4 window, host wall time per call."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import kernels, synth
from paper_2312_05385_b200.engine import serve_table
from paper_2312_05385_b200.graph import find_feasible_sites
prof = synth.config4_profile(); sites = find_feasible_sites(prof); a = synth.config4_window(1_000_000)
scores = np.ascontiguousarray(a.errs); cext = a.correct_ext()
serve = serve_table(sites, prof, 1); van = prof.model_latency(1)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
out = {}
ref = None
for name, (s, c) in {"pageable": (scores, cext),
                     "pinned": (torch.from_numpy(scores).pin_memory().numpy(),
                                torch.from_numpy(cext).pin_memory().numpy())}.items():
    for _ in range(2): kernels.eval_thresholds(s, c, serve, van, th, mode="hist")
    ts = []
    for _ in range(8):
        t0 = time.perf_counter(); kernels.eval_thresholds(s, c, serve, van, th, mode="hist"); ts.append(time.perf_counter() - t0)
    acc, sav = kernels.eval_thresholds(s, c, serve, van, th, mode="hist")
    ref = ref or (acc, sav)
    out[name] = {"ms": float(np.median(ts)) * 1e3, "candidates_per_s": 64 / float(np.median(ts)),
                 "same_results": bool(np.array_equal(acc, ref[0]) and np.array_equal(sav, ref[1]))}
print(json.dumps(out))
