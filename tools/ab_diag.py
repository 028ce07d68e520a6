"""A/B of diagonal-kernel variants on the config-4 window (CUDA-event time per sweep, L2 flushed)."""
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
ref = None
for ver in [int(v) for v in (sys.argv[1:] or ["1", "2", "3"])]:
    nat.set_diag_version(ver)
    h, o = sw.histograms(th) if hasattr(sw, "histograms") else (None, None)
    for _ in range(10): sw.evaluate_many(th, to_host=False)
    torch.cuda.synchronize(); nat.profile_read(); nat.profile_enable(True)
    for _ in range(100):
        (nat.l2_flush(flush) if os.environ.get("OWNFLUSH") else flush.zero_()); sw.evaluate_many(th, to_host=False)
    torch.cuda.synchronize(); nat.profile_enable(False)
    prof_ = nat.profile_read()
    acc, sav = sw.evaluate_many(th)
    if ref is None: ref = (acc, sav)
    same = bool(np.array_equal(acc, ref[0]) and np.array_equal(sav, ref[1]))
    print(json.dumps({"version": ver, "kernels": {k: v["ms"] / v["launches"] * 1e3 for k, v in prof_.items()}, "same_as_first": same}))
