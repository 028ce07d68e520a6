"""Where Algorithm 1's device loop spends its time: clock64 cycles per phase
(ee_tune_profile) for the 128- and 1000-record windows of tools/profile_tune.py."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_05385_b200 import synth, _native as nat
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import synthesize_workload
from paper_2312_05385_b200.tuner import TunerParams, tune
prof = synth.config4_profile(); s13 = find_feasible_sites(prof)
curve = {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(s13)}
ramps = [s13[0], s13[2], s13[4], s13[6], s13[8], s13[10]]
buf = torch.zeros(8, dtype=torch.int64, device="cuda")
for n in (128, 1000):
    recs = list(synthesize_workload(prof, n, 0.7, curve, seed=42, miscalibration=0.1).records)
    ev = WindowEvaluator(recs, ramps, prof)
    tune(recs, ramps, TunerParams(), prof, evaluator=ev)
    nat.check(nat.load_library().ee_tune_profile(nat.workspace(), buf.data_ptr()))
    res = tune(recs, ramps, TunerParams(), prof, evaluator=ev)
    nat.check(nat.load_library().ee_tune_profile(nat.workspace(), None))
    c = buf.cpu().numpy().astype(float)
    names = ["candidates", "scan", "fold", "select_tail", "update", "select_keys", "select_argmax"]
    print(json.dumps({"n": n, "us_at_1.965GHz": {k: round(v / 1965.0, 1) for k, v in zip(names, c)},
                      "total_us": round(c.sum() / 1965.0, 1)}))
