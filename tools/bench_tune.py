"""Config-1 style threshold tuning: tune() over a 1000-record x 6-ramp window,
GPU (device-resident Algorithm 1, and host loop) vs the reference CPU path
(oracle restatement over the compiled reference kernel). Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle as O
from paper_2312_05385_b200 import synth
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import synthesize_workload
from paper_2312_05385_b200.tuner import TunerParams, tune

prof = synth.config4_profile()
s13 = find_feasible_sites(prof)
curve = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(s13)}
w = synthesize_workload(prof, 1000, 0.7, curve, seed=42, miscalibration=0.1)
ramps = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
recs = list(w.records)
ev = WindowEvaluator(recs, ramps, prof)
out = {}
for name, dev in (("device_loop", True), ("host_loop", False)):
    for _ in range(3):
        res = tune(recs, ramps, TunerParams(), prof, evaluator=ev, device_loop=dev)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        res = tune(recs, ramps, TunerParams(), prof, evaluator=ev, device_loop=dev)
        ts.append(time.perf_counter() - t0)
    out[name] = {"ms_median": 1e3 * float(np.median(ts)), "rounds": res.rounds, "evals": res.evals}
# reference CPU path: Algorithm 1 over the compiled reference kernel (oracle/_ref) on a packed window
ref = O.reference_kernel()
scores, cext = O.pack_window(recs, ramps)
serve = O.serve_table(ramps, prof, 1)
van = prof.model_latency(1)
kern = ref if ref is not None else O
def ref_tune():
    return O.tune(recs, ramps, prof)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); ref_tune(); ts.append(time.perf_counter() - t0)
out["cpu_oracle_tune_ms_median_incl_packing"] = 1e3 * float(np.median(ts))
print(json.dumps(out))
