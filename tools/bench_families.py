"""Config-4 window, the other SURVEY §8d candidate families through the generic
path: C=768 axis sweep and C=65,536 random lattice rows (compute-ridge stress).
CUDA-event ms per evaluation (L2 flushed between). One JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites

prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
r = 12
lat = np.arange(64) / 63.0
fams = {"axis768": None, "random4096": lat[np.random.default_rng(1).integers(0, 64, size=(4096, r))],
        "random65536": lat[np.random.default_rng(1).integers(0, 64, size=(65536, r))]}
th = np.full((768, r), 0.3)
for j in range(r):
    th[j * 64:(j + 1) * 64, j] = lat
fams["axis768"] = th
sw = ShardedSweep(arrays, sites, prof)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for name, t in fams.items():
    reps = 3 if t.shape[0] > 10000 else 10
    sw.evaluate_many(t, to_host=False)
    torch.cuda.synchronize(); nat.profile_read(); nat.profile_enable(True)
    for _ in range(reps):
        flush.zero_(); sw.evaluate_many(t, to_host=False)
    torch.cuda.synchronize(); nat.profile_enable(False)
    p = nat.profile_read()
    ms = sum(v["ms"] for v in p.values()) / reps
    out[name] = {"candidates": int(t.shape[0]), "ms": ms, "candidates_per_s": t.shape[0] / (ms / 1e3),
                 "kernels": {k: v["ms"] / reps for k, v in p.items()}}
print(json.dumps(out))
