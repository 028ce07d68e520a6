import os, sys, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import synthesize_workload
from paper_2312_05385_b200.tuner import TunerParams, tune
prof = synth.config4_profile(); s13 = find_feasible_sites(prof)
curve = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(s13)}
ramps = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
for n in (128, 1000):
    recs = list(synthesize_workload(prof, n, 0.7, curve, seed=42, miscalibration=0.1).records)
    ev = WindowEvaluator(recs, ramps, prof)
    for _ in range(3): tune(recs, ramps, TunerParams(), prof, evaluator=ev)
    nat.profile_read(); nat.profile_enable(True)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); tune(recs, ramps, TunerParams(), prof, evaluator=ev); ts.append(time.perf_counter() - t0)
    nat.profile_enable(False)
    k = nat.profile_read()
    print(n, "wall_ms", 1e3 * np.median(ts), {a: b["ms"] / b["launches"] for a, b in k.items()})
