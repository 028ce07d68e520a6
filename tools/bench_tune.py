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

# grid_oracle (tuner.py:182-227) on the acceptance suite's instances
# (test_acceptance.py:52-67, its first 12: make_chain(8), 3 ramps, 64 records, step 0.01 ->
# a 101^3 = 1,030,301-point lattice): ours scores the lattice from its index on
# the device (ee_eval_lattice), the reference materialises it and runs its
# compiled kernel. Results must agree exactly.
from paper_2312_05385_b200.tuner import grid_oracle

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
ref_grid = None
if os.path.isdir(os.path.join(REF, "eesim")):
    sys.path.insert(0, REF)
    import eesim.graph as RG
    import eesim.trace as RT
    import eesim.tuner as RTu
    import eesim._kernels as RK
    ref_grid = RK.BACKEND
from paper_2312_05385_b200.graph import ModelProfile

nodes = [f"n{i}" for i in range(8)]  # make_chain(8)
lat = {x: {1: 10.0} for x in nodes}
rl = {x: {1: 0.5} for x in nodes[:-1]}
prof7 = ModelProfile(nodes, list(zip(nodes, nodes[1:])), lat, rl, nodes[-1])
s7 = find_feasible_sites(prof7)
g_ours, g_ref, agree = [], [], True
rng = np.random.default_rng(2024)
budget = TunerParams().acc_loss_budget
for seed in range(12):
    lo = float(rng.uniform(0.2, 0.5)); hi = float(rng.uniform(lo, 0.95))
    crv = {x.position: lo + (hi - lo) * i / 6 for i, x in enumerate(s7)}
    cont, mis = float(rng.uniform(0, 1)), float(rng.uniform(0, 0.4))
    rr = [s7[1], s7[3], s7[5]]
    recs = list(synthesize_workload(prof7, 64, cont, crv, seed=seed, miscalibration=mis).records)
    grid_oracle(recs, rr, budget, 0.01, prof7)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); go = grid_oracle(recs, rr, budget, 0.01, prof7); g_ours.append(time.perf_counter() - t0)
    if ref_grid is not None:
        rprof = RG.ModelProfile(nodes, list(zip(nodes, nodes[1:])), lat, rl, nodes[-1])
        rs = RG.find_feasible_sites(rprof)
        rw = RT.synthesize_workload(rprof, 64, cont, crv, seed=seed, miscalibration=mis)
        t0 = time.perf_counter()
        gr = RTu.grid_oracle(list(rw.records), [rs[1], rs[3], rs[5]], budget, 0.01, rprof)
        g_ref.append(time.perf_counter() - t0)
        agree &= dict(gr.thresholds) == dict(go.thresholds) and gr.savings_ms == go.savings_ms
out["grid_oracle"] = {
    "instances": 12, "lattice_points": 101 ** 3, "records": 64, "ramps": 3,
    "gpu_ms_median": 1e3 * float(np.median(g_ours)),
    "candidates_per_s": 101 ** 3 / float(np.median(g_ours)),
    "reference_cpu_ms_median": 1e3 * float(np.median(g_ref)) if g_ref else None,
    "reference_backend": ref_grid, "identical_results": bool(agree) if g_ref else None,
    "path": "tuner.grid_oracle -> WindowEvaluator.evaluate_lattice -> ee_eval_lattice (exact mode)"}
print(json.dumps(out))
