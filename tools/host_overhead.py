"""Host-side cost of one sweep call (no synchronisation): Python API vs raw C ABI."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites
prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
th = np.repeat((np.arange(64) / 63.0)[:, None], 12, axis=1)
sw = ShardedSweep(arrays, sites, prof)
ev = sw.local
out = {}
for name, fn in [("ShardedSweep.evaluate_many", lambda: sw.evaluate_many(th, to_host=False)),
                 ("torch.empty x3", lambda: [torch.empty(64, dtype=torch.float64, device="cuda") for _ in range(3)]),
                 ("event.record", lambda: torch.cuda.Event(enable_timing=True).record()),
                 ("flush.zero_", None)]:
    if fn is None:
        buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fn = buf.zero_
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    out[name] = (time.perf_counter() - t0) / 200 * 1e6
    torch.cuda.synchronize()
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
