"""Config-4 window, the C = 768 axis family (base 0.3, ramp j swept over 64
points): k_axis vs the generic SWAR path, per sweep (CUDA events, L2 flushed)
and in a stream of sweeps (one CUDA graph)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.distributed import ShardedSweep
from paper_2312_05385_b200.graph import find_feasible_sites

prof = synth.config4_profile(); sites = find_feasible_sites(prof); arrays = synth.config4_window(1_000_000)
r = 12
th = np.full((768, r), 0.3)
for j in range(r):
    th[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
sw = ShardedSweep(arrays, sites, prof)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
ref = None
for name, special in (("k_axis", True), ("generic", False)):
    nat.set_special(special)
    acc, sav = sw.evaluate_many(th)
    if ref is None:
        ref = (acc, sav)
    out[name] = {"identical": bool(np.array_equal(acc, ref[0]) and np.array_equal(sav, ref[1]))}
    for _ in range(3): sw.evaluate_many(th, to_host=False)
    nat.profile_read(); nat.profile_enable(True)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); sw.evaluate_many(th, to_host=False); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    nat.profile_enable(False)
    kern = nat.profile_read()
    out[name]["sweep_ms_median"] = float(np.median(ts))
    out[name]["kernels_ms_per_sweep"] = {k: v["ms"] / 20 for k, v in kern.items()}
    K = 50
    if special:  # the generic path stages tables through pinned memory: not capturable
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(K): sw.evaluate_many(th, to_host=False)
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        out[name]["stream_ms_per_sweep"] = ms
        del g
    else:
        ms = out[name]["sweep_ms_median"]
    out[name]["candidates_per_s"] = 768 / (ms / 1e3)
    print(name, json.dumps(out[name]), flush=True)
nat.set_special(True)
print(json.dumps(out))
