"""Algorithm 1 (tuner.tune, §8 A7): the device-resident hill climb vs the
reference's CPU path (Algorithm 1 over the reference's compiled Cython kernel,
oracle/_ref, packing the window per call as engine.WindowEvaluator does), on
the default 128-record tuning history and config 1's 1,000-record window.
Thresholds must agree bit for bit. One JSON line."""
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
ramps = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
ref = O.reference_kernel()
out = {"cpu_kind": "reference (oracle/_ref Cython)" if ref is not None else "port (C oracle)"}
for n in (128, 1000):
    recs = list(synthesize_workload(prof, n, 0.7, curve, seed=42, miscalibration=0.1).records)

    def ours():
        return tune(recs, ramps, TunerParams(), prof)  # packs + uploads the window, one launch

    ev = WindowEvaluator(recs, ramps, prof)
    for _ in range(3):
        res = ours()
    torch.cuda.synchronize()
    ts, tr = [], []
    for _ in range(20):
        t0 = time.perf_counter(); res = ours(); ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter(); tune(recs, ramps, TunerParams(), prof, evaluator=ev); tr.append(time.perf_counter() - t0)
    tc = []
    for _ in range(10):
        t0 = time.perf_counter(); th, *_ = O.tune(recs, ramps, prof, kernel=ref); tc.append(time.perf_counter() - t0)
    out[f"n{n}"] = {"gpu_tune_ms": 1e3 * float(np.median(ts)),
                    "gpu_tune_resident_window_ms": 1e3 * float(np.median(tr)),
                    "cpu_reference_tune_ms": 1e3 * float(np.median(tc)),
                    "rounds": res.rounds, "evals": res.evals,
                    "bit_identical_thresholds": res.threshold_vector(ramps) == th}
print(json.dumps(out))
