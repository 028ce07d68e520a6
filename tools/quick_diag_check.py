import sys, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_gpu_parity import random_window
from oracle import oracle as O
from paper_2312_05385_b200 import kernels
for n, r in [(5000, 12), (1000, 16), (40000, 14), (1, 2)]:
    rng = np.random.default_rng(n)
    scores, cext, serve, vanilla, _ = random_window(rng, n, r, 1)
    th = np.repeat((np.arange(64) / 63.0)[:, None], r, axis=1)
    acc, sav = kernels.eval_thresholds(scores, cext, serve, vanilla, th, mode="hist")
    ao, so = O.eval_thresholds(scores, cext, serve, vanilla, th)
    print(n, r, np.array_equal(acc, ao), np.allclose(sav, so, rtol=1e-9, atol=1e-12), flush=True)
