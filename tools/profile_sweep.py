"""Run a few config-4 sweeps for ncu (kernel capture) — not a benchmark."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2312_05385_b200 import synth
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites

family = sys.argv[1] if len(sys.argv) > 1 else "diagonal"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prof = synth.config4_profile()
sites = find_feasible_sites(prof)
arrays = synth.config4_window(1_000_000)
r = 12
if family == "diagonal":
    th = np.repeat((np.arange(64) / 63.0)[:, None], r, axis=1)
elif family == "axis":
    th = np.full((768, r), 0.3)
    for j in range(r):
        th[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
else:
    th = (np.arange(64) / 63.0)[np.random.default_rng(1).integers(0, 64, size=(64, r))]
sw = ShardedSweep(arrays, sites, prof)
if os.environ.get("DIAG_VERSION"):
    from paper_2312_05385_b200 import _native
    _native.set_diag_version(int(os.environ["DIAG_VERSION"]))
for _ in range(reps):
    sw.evaluate_many(th, to_host=False)
torch.cuda.synchronize()
print("done", family)
