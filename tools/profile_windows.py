"""K config-4 windows as one persistent sweep (distributed.WindowStream over 4
resident copies of the 1M x 12 window), for an ncu capture of
k_diag3_windows_db (not a benchmark). Usage: profile_windows.py [K]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth
from paper_2312_05385_b200.distributed import ShardedSweep, WindowStream
from paper_2312_05385_b200.graph import find_feasible_sites

k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sweeps = [ShardedSweep(arrays, sites, prof) for _ in range(4)]
ws = WindowStream(sweeps, order=[i % 4 for i in range(k)])
for _ in range(3):
    ws.run(th)
torch.cuda.synchronize()
print("done", k)
