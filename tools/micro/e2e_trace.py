"""EEB200_TRACE_HOST=1 run of the drop-in call (host timestamps per step)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2312_05385_b200 import kernels, synth
from paper_2312_05385_b200.engine import serve_table
from paper_2312_05385_b200.graph import find_feasible_sites
prof = synth.config4_profile(); sites = find_feasible_sites(prof)[:12]
arrays = synth.config4_window(1_000_000)
scores = torch.from_numpy(np.ascontiguousarray(arrays.errs)).pin_memory().numpy()
cext = torch.from_numpy(arrays.correct_ext()).pin_memory().numpy()
serve = serve_table(sites, prof, 1); vanilla = prof.model_latency(1)
g = np.linspace(0.0, 1.0, 64); th = np.repeat(g[:, None], 12, axis=1).copy()
for _ in range(6):
    t0 = time.perf_counter(); kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode="hist")
    print(f"python call {1e6 * (time.perf_counter() - t0):.1f} us", file=sys.stderr)

# the native entry point alone (no Python wrapper), same buffers
import ctypes
from paper_2312_05385_b200 import _native as nat
lib = nat.load_library()
acc = np.empty(64); sav = np.empty(64)
st = nat.stream_handle(torch); ws = nat.workspace()
for _ in range(4):
    t0 = time.perf_counter()
    nat.check(lib.ee_eval_thresholds_host(ws, scores.ctypes.data, cext.ctypes.data, 1_000_000, 12,
                                          serve.ctypes.data, float(vanilla), th.ctypes.data, 64, 2,
                                          acc.ctypes.data, sav.ctypes.data, 0, st))
    print(f"direct native call {1e6 * (time.perf_counter() - t0):.1f} us", file=sys.stderr)
