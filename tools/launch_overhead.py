"""Fixed per-launch cost of k_diag2 seen by CUDA events: tiny windows vs the 1M window."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import WindowArrays
from paper_2312_05385_b200 import synth
prof = synth.config4_profile(); sites = find_feasible_sites(prof)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
res = {}
for n in [32, 32 * 32 * 148, 1_000_000]:
    a = synth.config4_window(n)
    ev = WindowEvaluator.from_arrays(a, sites, prof, mode="hist")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(10): ev._eval_device(th)
    torch.cuda.synchronize(); nat.profile_read(); nat.profile_enable(True)
    for _ in range(50):
        flush.zero_(); ev._eval_device(th)
    torch.cuda.synchronize(); nat.profile_enable(False)
    p = nat.profile_read()
    res[n] = {k: round(v["ms"] / v["launches"] * 1e3, 2) for k, v in p.items()}
print(json.dumps(res))
