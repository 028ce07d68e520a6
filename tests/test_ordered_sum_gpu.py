"""osum::warp_ordered_sum (the fold of ee_tune) against the plain sequential
fp64 chain, bit for bit, on the inputs that break naive reordering: binade
crossings, exact ties at the running grid, zeros, tiny and huge addends,
repeated values (serve tables) and long rows."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2312_05385_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _seq(row):
    s = 0.0
    for v in row:
        s = float(np.float64(s) + np.float64(v))
    return s


def _rows(rng):
    rows = []
    serve = np.sort(rng.uniform(1.0, 20.0, size=13))
    rows.append(serve[rng.integers(0, 13, size=1000)])           # a tune fold
    rows.append(serve[rng.integers(0, 13, size=20000)])
    rows.append(np.full(3000, 0.1))                              # repeating binary fraction
    rows.append(np.full(5000, 1.5))                              # exact ties once the sum is large
    rows.append(np.full(777, 2.0 ** -20 * 3))                    # ties at small scale
    rows.append(np.concatenate([[1e-300], np.full(300, 1.0)]))   # tiny start
    rows.append(np.concatenate([np.zeros(50), rng.uniform(0, 1, 400)]))
    rows.append(np.concatenate([rng.uniform(0, 1, 200), [1e15], rng.uniform(0, 1, 200)]))  # big jump
    rows.append(rng.uniform(0, 1, 1) * 0 + rng.uniform(0, 1e-3, 129))
    tie = np.full(4096, 1.0)
    tie[::7] = 1.0 + 2.0 ** -40                                  # ties appear as the sum grows
    rows.append(tie)
    rows.append(np.array([]))
    rows.append(np.array([3.25]))
    return rows


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_warp_ordered_sum_is_the_sequential_chain(cuda, seed):
    rng = np.random.default_rng(seed)
    lib = nat.load_library()
    for row in _rows(rng):
        n = row.size
        d = torch.tensor(row, dtype=torch.float64, device="cuda").reshape(1, n)
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        nat.check(lib.ee_sequential_sum(d.data_ptr() if n else None, n, 1, out.data_ptr(),
                                        nat.stream_handle(torch)))
        got = float(out.item())
        want = _seq(row)
        assert got == want or (np.isnan(got) and np.isnan(want)), (n, row[:4], got, want)


def test_many_rows(cuda):
    rng = np.random.default_rng(9)
    serve = rng.uniform(0.5, 30.0, size=8)
    vals = serve[rng.integers(0, 8, size=(64, 1500))]
    d = torch.tensor(vals, device="cuda")
    out = torch.empty(64, dtype=torch.float64, device="cuda")
    nat.check(nat.load_library().ee_sequential_sum(d.data_ptr(), 1500, 64, out.data_ptr(),
                                                   nat.stream_handle(torch)))
    got = out.cpu().numpy()
    for i in range(64):
        assert got[i] == _seq(vals[i])
