"""Where the drop-in call's 2.1 ms goes (config-4 window, pinned inputs): the
whole kernels.eval_thresholds call vs the host pack of correct_ext alone vs the
96 MB score H2D alone."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2312_05385_b200 import kernels, synth, _native as nat
from paper_2312_05385_b200.engine import serve_table
from paper_2312_05385_b200.graph import find_feasible_sites

prof = synth.config4_profile()
sites = find_feasible_sites(prof)[:12]
arrays = synth.config4_window(1_000_000)
scores = torch.from_numpy(np.ascontiguousarray(arrays.errs)).pin_memory().numpy()
cext = torch.from_numpy(arrays.correct_ext()).pin_memory().numpy()
serve = serve_table(sites, prof, 1); vanilla = prof.model_latency(1)
g = np.linspace(0.0, 1.0, 64)
th = np.repeat(g[:, None], 12, axis=1).copy()
lib = nat.load_library()
bits = torch.empty(1_000_000, dtype=torch.int32).pin_memory()
d = torch.empty(scores.nbytes, dtype=torch.uint8, device="cuda")
hs = torch.from_numpy(scores.view(np.uint8).reshape(-1))

def med(fn, k=15):
    for _ in range(3): fn()
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))

out = {
    "call_ms": med(lambda: kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode="hist")),
    "pack_ms_all_cores": med(lambda: nat.check(lib.ee_pack_correct_host(cext.ctypes.data, 1_000_000, 13, bits.data_ptr(), 0))),
    "h2d_scores_ms": med(lambda: d.copy_(hs, non_blocking=True)),
    "cores": os.cpu_count(),
}
print(json.dumps(out))

# the two together, as the call overlaps them: H2D issued, then the host pack
def both():
    d.copy_(hs, non_blocking=True)
    nat.check(lib.ee_pack_correct_host(cext.ctypes.data, 1_000_000, 13, bits.data_ptr(), 0))
print(json.dumps({"h2d_and_pack_overlapped_ms": med(both)}))
