import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_parity import random_window
from conftest import make_chain
from oracle import oracle as O
from paper_2312_05385_b200 import _native
from paper_2312_05385_b200.engine import WindowEvaluator
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import WindowArrays
def case(r, n, m, c_rep, mods):
    rng = np.random.default_rng(9100 + r + n)
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1, nan_frac=0.01)
    a=scores.copy()
    scores[rng.random((n, r)) < 0.01] = np.inf
    scores[rng.random((n, r)) < 0.01] = -0.0
    cext[:, r] = (rng.random(n) < 0.8).astype(np.float64)
    extra = np.array([0.0, np.inf, -np.inf, 1.0])
    vals = np.unique(np.concatenate([np.round(rng.random(4 * m) * 997) / 997, extra]))[:m]
    rows = np.repeat(np.concatenate([vals, [np.nan]]), c_rep); rng.shuffle(rows)
    if 'nonan' in mods: scores[np.isnan(scores)] = 0.3
    if 'noinf' in mods: scores[np.isinf(scores)] = 0.4
    if 'c1' in mods: cext[:, r] = 1
    th = np.repeat(rows[:, None], r, axis=1)
    arrays = WindowArrays(scores, cext.astype(np.uint8))
    prof = make_chain(r + 1)
    ev = WindowEvaluator.from_arrays(arrays, find_feasible_sites(prof)[:r], prof, mode="hist")
    h2, o2 = ev.histograms(th)
    ho, oo = O.eval_hist(scores, cext, th)
    bad = np.argwhere(h2 != ho)
    print(r, n, m, mods, "hist mismatches", len(bad), "ok mism", int((o2 != oo).sum()), "vals[:5]", vals[:5], "max", vals.max())
    for c, s in bad[:6]:
        print("   cand", c, "th", rows[c], "site", s, "got", h2[c, s], "want", ho[c, s])
for mods in [(), ('nonan',), ('noinf',), ('c1',), ('nonan','noinf','c1')]:
    case(12, 70001, 64, 1, mods)
case(12, 4099, 64, 1, ())
case(12, 70001, 40, 1, ())
