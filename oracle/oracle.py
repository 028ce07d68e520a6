"""CPU oracle for the early-exit decision path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module, and only as the checker or the timed CPU baseline.
The product package (paper_2312_05385_b200) never imports it.

Contents, each a restatement of the reference (paths under /root/reference):
  * C kernels from exitcore_oracle.c via ctypes:
      exit_sites            pkg/src/eesim/_kernels/_exitcore.pyx:11-24
      eval_thresholds       pkg/src/eesim/_kernels/_exitcore.pyx:27-56
      eval_hist             integer histogram implied by the same loop
      decision_scores       pkg/src/eesim/engine.py:106-121
  * pure-Python restatements:
      serve_table           pkg/src/eesim/engine.py:124-132
      pack_window           pkg/src/eesim/engine.py:152-163
      brute_window          pkg/tests/conftest.py:103-136 (plain walk over ramps)
      tune                  pkg/src/eesim/tuner.py:97-171 (Algorithm 1)
      grid_oracle           pkg/src/eesim/tuner.py:182-227
      exit_record           pkg/src/eesim/engine.py:189-220
  * reference_kernel(): the reference's own Cython kernel compiled from
    /root/reference by oracle/Makefile into oracle/_ref/ (when present).
Pinned against the reference's golden vectors by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_exit_sites.argtypes = [vp, i64, i32, vp, vp]
        L.oracle_eval_thresholds.argtypes = [vp, vp, i64, i32, vp, f64, vp, i64, vp, vp]
        L.oracle_eval_hist.argtypes = [vp, vp, i64, i32, vp, i64, vp, vp]
        L.oracle_decision_scores.argtypes = [vp, i64, i32, i32, vp]
        for f in (L.oracle_exit_sites, L.oracle_eval_thresholds, L.oracle_eval_hist,
                  L.oracle_decision_scores):
            f.restype = None
        _lib = L
    return _lib


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def exit_sites(scores, thresholds) -> np.ndarray:
    scores, thresholds = _c(scores), _c(thresholds)
    n, r = scores.shape
    out = np.empty(n, dtype=np.int64)
    lib().oracle_exit_sites(scores.ctypes.data, n, r, thresholds.ctypes.data, out.ctypes.data)
    return out


def eval_thresholds(scores, correct_ext, serve, vanilla, thresholds):
    scores, correct_ext, serve, thresholds = _c(scores), _c(correct_ext), _c(serve), _c(thresholds)
    n, r = scores.shape
    c = thresholds.shape[0]
    acc, sav = np.empty(c), np.empty(c)
    lib().oracle_eval_thresholds(scores.ctypes.data, correct_ext.ctypes.data, n, r,
                                 serve.ctypes.data, float(vanilla), thresholds.ctypes.data, c,
                                 acc.ctypes.data, sav.ctypes.data)
    return acc, sav


def eval_hist(scores, correct_ext, thresholds):
    scores, correct_ext, thresholds = _c(scores), _c(correct_ext), _c(thresholds)
    n, r = scores.shape
    c = thresholds.shape[0]
    hist = np.empty((c, r + 1), dtype=np.int64)
    ok = np.empty(c, dtype=np.int64)
    lib().oracle_eval_hist(scores.ctypes.data, correct_ext.ctypes.data, n, r,
                           thresholds.ctypes.data, c, hist.ctypes.data, ok.ctypes.data)
    return hist, ok


def decision_scores(errs, k: int):
    errs = _c(errs)
    if k <= 1 or errs.shape[1] <= 1:
        return errs
    n, r = errs.shape
    out = np.empty_like(errs)
    lib().oracle_decision_scores(errs.ctypes.data, n, r, k, out.ctypes.data)
    return out


def serve_table(sites, profile, batch: int) -> np.ndarray:
    r = len(sites)
    serve = np.empty(r + 1)
    acc = 0.0
    for j, s in enumerate(sites):
        acc += s.ramp_ms(batch)
        serve[j] = s.prefix_ms(batch) + acc
    serve[r] = profile.model_latency(batch) + acc if r else profile.model_latency(batch)
    return serve


def pack_window(records, sites, k: int = 1):
    """(scores, correct_ext) exactly as WindowEvaluator builds them."""
    n, r = len(records), len(sites)
    errs = np.empty((n, r))
    cext = np.ones((n, r + 1))
    for i, rec in enumerate(records):
        for j, s in enumerate(sites):
            sig = rec.ramp_signals[s.position]
            errs[i, j] = sig.err
            cext[i, j] = 1.0 if sig.label == rec.final_label else 0.0
    return decision_scores(errs, k), cext


def exit_record(record, active, profile, batch: int = 1, k: int = 1):
    """(exit position or None, released label, correct, serve ms)."""
    acc = 0.0
    window = []
    for site, threshold in active:
        acc += site.ramp_ms(batch)
        err = record.ramp_signals[site.position].err
        window.append(err)
        if len(window) > k:
            window.pop(0)
        score = err if k <= 1 else sum(window) / len(window)
        if score < threshold:
            label = record.ramp_signals[site.position].label
            return site.position, label, label == record.final_label, site.prefix_ms(batch) + acc
    return None, record.final_label, True, profile.model_latency(batch) + acc


def brute_window(records, active, profile, k: int = 1):
    vanilla = profile.model_latency(1)
    ok, sav = 0, 0.0
    exits = {s.position: 0 for s, _ in active}
    for rec in records:
        pos, _, correct, serve = exit_record(rec, active, profile, 1, k)
        ok += correct
        sav += vanilla - serve
        if pos is not None:
            exits[pos] += 1
    n = len(records)
    return ok / n, sav / n, {p: c / n for p, c in exits.items()}


def tune(records, ramps, profile, budget=0.01, init_step=0.1, min_step=0.01, k=1, kernel=None):
    """Algorithm 1 (tuner.py:97-171) over the C oracle kernel, or over `kernel`
    (any module with the `_kernels` eval_thresholds signature, e.g. the
    reference's compiled Cython backend); returns (thresholds, sav, acc,
    rounds, evals, trace)."""
    eval_thresholds_ = kernel.eval_thresholds if kernel is not None else eval_thresholds
    if not ramps:
        return [], 0.0, 1.0, 0, 0, ()
    scores, cext = pack_window(records, ramps, k)
    serve = serve_table(ramps, profile, 1)
    vanilla = profile.model_latency(1)
    r = len(ramps)
    th = np.zeros(r)
    steps = np.full(r, init_step)
    floor = 1.0 - budget
    a, s = eval_thresholds_(scores, cext, serve, vanilla, th.reshape(1, r))
    acc_cur, sav_cur = float(a[0]), float(s[0])
    rounds, evals, trace = 0, 1, [tuple(steps)]
    while True:
        rounds += 1
        elig = [i for i in range(r) if th[i] < 1.0]
        if not elig:
            break
        rows = np.repeat(th.reshape(1, r), len(elig), axis=0)
        for p, i in enumerate(elig):
            rows[p, i] = min(1.0, th[i] + steps[i])
        accs, savs = eval_thresholds_(scores, cext, serve, vanilla, rows)
        evals += len(elig)
        best, best_key, viol = None, None, []
        for p, i in enumerate(elig):
            if accs[p] < floor - 1e-12:
                viol.append(i)
                continue
            dsav = float(savs[p]) - sav_cur
            dloss = acc_cur - float(accs[p])
            key = (1, dsav, -i) if dloss <= 1e-12 else (0, dsav / dloss, dsav, -i)
            if best_key is None or key > best_key:
                best_key, best = key, p
        if best is not None:
            i = elig[best]
            th[i] = min(1.0, th[i] + steps[i])
            acc_cur, sav_cur = float(accs[best]), float(savs[best])
            steps[i] *= 2.0
        elif all(steps[i] <= min_step + 1e-12 for i in elig):
            break
        for i in viol:
            steps[i] = max(min_step, steps[i] / 2.0)
        trace.append(tuple(steps))
    return [float(t) for t in th], sav_cur, acc_cur, rounds, evals, tuple(trace)


def lattice(step: float) -> np.ndarray:
    count = int(np.floor(1.0 / step + 1e-9)) + 1
    vals = np.minimum(np.arange(count) * step, 1.0)
    if vals[-1] < 1.0 - 1e-12:
        vals = np.append(vals, 1.0)
    return vals


def grid_oracle(records, ramps, profile, budget, step, k=1):
    """(thresholds, sav, acc, n_points) by exhaustive C-oracle evaluation."""
    vals = lattice(step)
    r = len(ramps)
    grids = np.meshgrid(*([vals] * r), indexing="ij")
    rows = np.stack([g.ravel() for g in grids], axis=1)
    scores, cext = pack_window(records, ramps, k)
    accs, savs = eval_thresholds(scores, cext, serve_table(ramps, profile, 1),
                                 profile.model_latency(1), rows)
    feas = np.flatnonzero(accs >= (1.0 - budget) - 1e-12)
    best = feas[np.argmax(savs[feas])]
    return [float(t) for t in rows[best]], float(savs[best]), float(accs[best]), len(rows)


def reference_kernel():
    """The reference's own compiled Cython kernel module (oracle/_ref), or None."""
    paths = glob.glob(os.path.join(REF_DIR, "_exitcore*.so"))
    if not paths:
        return None
    spec = importlib.util.spec_from_file_location("_exitcore", paths[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
