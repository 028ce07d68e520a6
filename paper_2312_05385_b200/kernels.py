"""Drop-in replacement for the reference module `eesim._kernels`.

Reference seam: pkg/src/eesim/_kernels/__init__.py:14-48 exposes
`eval_thresholds`, `exit_sites`, `BACKEND`, `get_backend(name)` and
`available_backends()`; the engine looks the two callables up on every call
(pkg/src/eesim/engine.py:168,177), so assigning these functions onto that
module (see `install_into`) swaps the B200 kernels in.

Differences from the reference, all deliberate:
  * one backend ("cuda"); no numpy fallback and no env-var dispatch;
  * shapes are checked (the Cython kernel reads out of bounds on a short
    threshold vector) and mismatches raise `ParameterError`;
  * `correct_ext` must hold 0.0/1.0 only (the engine never builds anything
    else, engine.py:159) — other values raise ValueError;
  * inputs may also be CUDA torch tensors, in which case nothing is copied
    across PCIe and torch tensors come back.
Argument types and errors otherwise follow the Cython typed memoryviews
(`double[:, ::1]`, `double[::1]`): lists raise TypeError, wrong dtype /
rank / non-C-contiguous raise ValueError.
"""

from __future__ import annotations

import os
import sys

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError

BACKEND = "cuda"

_CY_NAMES = {"int64": "long", "int32": "int", "float32": "float", "float16": "half",
             "bool": "bool", "uint8": "unsigned char"}


def get_backend(name: str):
    """Return the kernel module for `name`; only "cuda" exists here."""
    if name == "cuda":
        return sys.modules[__name__]
    raise ValueError(f"unknown kernel backend {name!r}")


def available_backends() -> list[str]:
    return ["cuda"]


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _check_view(x, ndim: int, what: str):
    """Validate like a Cython `double[...:, ::1]` memoryview; returns ndarray or tensor."""
    if _is_cuda_tensor(x):
        import torch

        if x.dtype != torch.float64:
            raise ValueError(f"Buffer dtype mismatch, expected 'double' but got {x.dtype} ({what})")
        if x.dim() != ndim:
            raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {x.dim()})")
        if not x.is_contiguous():
            raise ValueError("tensor is not C-contiguous")
        return x
    if not isinstance(x, np.ndarray):
        if isinstance(x, (bytes, bytearray, memoryview)):
            x = np.asarray(memoryview(x))
        else:
            raise TypeError(f"a bytes-like object is required, not '{type(x).__name__}'")
    if x.dtype != np.float64:
        got = _CY_NAMES.get(x.dtype.name, x.dtype.name)
        raise ValueError(f"Buffer dtype mismatch, expected 'double' but got '{got}'")
    if x.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {x.ndim})")
    if not x.flags.c_contiguous:
        raise ValueError("ndarray is not C-contiguous")
    return x


def _mode_code(mode: str | None) -> int:
    mode = mode or os.environ.get("EEB200_MODE", "auto")
    try:
        return nat.MODES[mode]
    except KeyError:
        raise ParameterError(f"unknown evaluation mode {mode!r} (auto, exact, hist)") from None


def _to_device(torch, x):
    if _is_cuda_tensor(x):
        return x
    t = torch.from_numpy(x)
    return t.to("cuda", non_blocking=t.is_pinned())


def pack_correct_host(correct_ext, n_threads: int = 0) -> np.ndarray:
    """correct_ext f64 (N, R+1) -> u32 bit rows, packed on the host CPU cores
    (ValueError if an entry is not exactly 0.0 or 1.0)."""
    correct_ext = _check_view(correct_ext, 2, "correct_ext")
    n, r1 = correct_ext.shape
    bits = np.empty(n, dtype=np.uint32)
    nat.check(nat.load_library().ee_pack_correct_host(
        correct_ext.ctypes.data if n else None, n, r1, bits.ctypes.data if n else None,
        int(n_threads)))
    return bits


def pack_correct(correct_ext, torch=None):
    """correct_ext f64 (N, R+1) -> (u32 bit rows on device, device flag)."""
    torch = torch or nat.torch_cuda()
    lib = nat.load_library()
    n, r1 = correct_ext.shape
    if r1 - 1 > nat.MAX_RAMPS:
        raise ParameterError(f"{r1 - 1} ramps exceed the supported maximum of {nat.MAX_RAMPS}")
    d = _to_device(torch, correct_ext)
    bits = torch.empty(n, dtype=torch.int32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.check(lib.ee_pack_correct(nat.ptr(d), n, r1, nat.ptr(bits), flag.data_ptr(),
                                  nat.stream_handle(torch)))
    return bits, flag


def exit_sites(scores, thresholds):
    """Per-record exit index for one config; R means no exit.

    Replaces _exitcore.exit_sites (_exitcore.pyx:11-24)."""
    scores = _check_view(scores, 2, "scores")
    thresholds = _check_view(thresholds, 1, "thresholds")
    n, r = scores.shape
    if thresholds.shape[0] != r:
        raise ParameterError(f"thresholds has {thresholds.shape[0]} entries for {r} ramps")
    torch = nat.torch_cuda()
    lib = nat.load_library()
    d_s = _to_device(torch, scores)
    d_t = _to_device(torch, thresholds)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    nat.check(lib.ee_exit_sites(nat.ptr(d_s), n, r, nat.ptr(d_t), nat.ptr(out),
                                nat.stream_handle(torch)))
    if _is_cuda_tensor(scores):
        return out
    return out.cpu().numpy()


def eval_thresholds(scores, correct_ext, serve, vanilla, thresholds, *, mode: str | None = None):
    """(accuracy, mean savings) for each row of a (C, R) threshold matrix.

    Replaces _exitcore.eval_thresholds (_exitcore.pyx:27-56). `mode`:
    "exact" reproduces the Cython accumulation order bit for bit; "hist"
    reduces exact integer histograms (acc bit-identical, savings correctly
    rounded); "auto" (default) picks exact up to 4096 samples.
    """
    scores = _check_view(scores, 2, "scores")
    correct_ext = _check_view(correct_ext, 2, "correct_ext")
    serve = np.ascontiguousarray(serve.cpu().numpy() if _is_cuda_tensor(serve) else serve)
    serve = _check_view(serve, 1, "serve")
    on_device = _is_cuda_tensor(thresholds) or _is_cuda_tensor(scores)
    if _is_cuda_tensor(thresholds):
        thresholds = thresholds.cpu().numpy()
    thresholds = _check_view(thresholds, 2, "thresholds")
    n, r = scores.shape
    c = thresholds.shape[0]
    if tuple(correct_ext.shape) != (n, r + 1):
        raise ParameterError(f"correct_ext shape {tuple(correct_ext.shape)} != ({n}, {r + 1})")
    if serve.shape[0] != r + 1:
        raise ParameterError(f"serve has {serve.shape[0]} entries, expected {r + 1}")
    if thresholds.shape[1] != r:
        raise ParameterError(f"thresholds have {thresholds.shape[1]} columns for {r} ramps")
    if r > nat.MAX_RAMPS:
        raise ParameterError(f"{r} ramps exceed the supported maximum of {nat.MAX_RAMPS}")
    code = _mode_code(mode)
    torch = nat.torch_cuda()
    lib = nat.load_library()
    if not _is_cuda_tensor(scores) and not _is_cuda_tensor(correct_ext):
        # host buffers (the reference's calling convention): one native call packs
        # correct_ext on the CPU cores while the scores stream to the device
        acc = np.empty(c)
        sav = np.empty(c)
        nat.check(lib.ee_eval_thresholds_host(
            nat.workspace(), scores.ctypes.data if scores.size else None,
            correct_ext.ctypes.data if correct_ext.size else None, n, r, serve.ctypes.data,
            float(vanilla), thresholds.ctypes.data if thresholds.size else None, c, code,
            acc.ctypes.data, sav.ctypes.data, 0, nat.stream_handle(torch)))
        return acc, sav
    d_s = _to_device(torch, scores)
    bits, flag = pack_correct(correct_ext, torch)
    acc = torch.empty(c, dtype=torch.float64, device="cuda")
    sav = torch.empty(c, dtype=torch.float64, device="cuda")
    nat.check(lib.ee_eval_thresholds(
        nat.workspace(), nat.ptr(d_s), nat.ptr(bits), n, r, serve.ctypes.data, float(vanilla),
        thresholds.ctypes.data if thresholds.size else None, c, code, None, None,
        nat.ptr(acc), nat.ptr(sav), nat.stream_handle(torch)))
    if n and int(flag.item()):
        raise ValueError("correct_ext must contain only 0.0 and 1.0")
    if on_device:
        return acc, sav
    return acc.cpu().numpy(), sav.cpu().numpy()


def _reraise_as(errors_mod, fn):
    """Wrap `fn` so this package's EESimError subclasses surface as the same-named
    classes of the target package's `errors` module (a reference
    caller's `except eesim.errors.ParameterError` must still catch them)."""
    import functools

    from paper_2312_05385_b200 import errors as ours

    names = ("ParameterError", "GridCapError", "ValidationError", "GraphError")

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        try:
            return fn(*args, **kw)
        except ours.EESimError as exc:
            for name in names:
                if isinstance(exc, getattr(ours, name)) and hasattr(errors_mod, name):
                    raise getattr(errors_mod, name)(*exc.args) from exc
            raise

    return wrapper


def install_into(module) -> None:
    """Swap these kernels into a reference `eesim._kernels` module object.

    engine.py resolves `_kernels.eval_thresholds` / `_kernels.exit_sites` at
    call time (engine.py:168,177), so after this every WindowEvaluator — and
    therefore tune, grid_oracle, evaluate_window and ramp adjustment — runs
    on the GPU. When the target package has an `errors` module (eesim.errors,
    pkg/src/eesim/errors.py:4-21), shape errors are raised as ITS classes."""
    import importlib

    errors_mod = None
    name = getattr(module, "__name__", "")
    pkg = name.rsplit(".", 1)[0] if isinstance(name, str) and "." in name else ""
    if pkg:
        try:
            errors_mod = importlib.import_module(pkg + ".errors")
        except ImportError:
            errors_mod = None
    if errors_mod is None:
        module.eval_thresholds = eval_thresholds
        module.exit_sites = exit_sites
    else:
        module.eval_thresholds = _reraise_as(errors_mod, eval_thresholds)
        module.exit_sites = _reraise_as(errors_mod, exit_sites)
    module.BACKEND = BACKEND


def classify_candidates(thresholds):
    """Which sweep family a (C, R) candidate matrix belongs to, as the native
    dispatch sees it (host only, no device work): ("diagonal", m, None),
    ("axis", m, base vector) or ("generic", 0, None); m = distinct values."""
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    if th.ndim != 2:
        raise ParameterError(f"thresholds must be 2-D, got {th.shape}")
    c, r = th.shape
    import ctypes

    kind = ctypes.c_int32()
    m = ctypes.c_int32()
    base = np.empty(max(r, 1))
    nat.check(nat.load_library().ee_classify_candidates(
        th.ctypes.data if th.size else None, c, r, ctypes.byref(kind), ctypes.byref(m),
        base.ctypes.data))
    if kind.value == 1:
        return "diagonal", m.value, None
    if kind.value == 2:
        return "axis", m.value, base[:r].copy()
    return "generic", 0, None


def eval_thresholds_windows(evaluators, thresholds, order=None):
    """acc, sav [len(order), C] (CUDA f64) for diagonal candidate rows over many
    resident windows at once (ee_eval_thresholds_windows: one persistent sweep
    launch + one finalisation). `evaluators` are WindowEvaluators with the same
    n, r, serve table and vanilla latency; `order` lists which evaluator each
    output row sweeps (default: each once)."""
    torch = nat.torch_cuda()
    th = np.ascontiguousarray(thresholds, dtype=np.float64)
    evs = list(evaluators)
    if not evs:
        raise ParameterError("no windows")
    e0 = evs[0]
    for e in evs[1:]:
        if e.n != e0.n or e.r != e0.r or not np.array_equal(e.serve, e0.serve) or e.vanilla_ms != e0.vanilla_ms:
            raise ParameterError("windows must share n, r, serve table and vanilla latency")
    order = list(range(len(evs))) if order is None else [int(i) for i in order]
    if not order:
        raise ParameterError("empty window order")
    if any(i < 0 or i >= len(evs) for i in order):
        raise ParameterError(f"window order entries must lie in [0, {len(evs)})")
    if th.ndim != 2 or th.shape[1] != e0.r:
        raise ParameterError(f"thresholds must be (C, {e0.r}), got {th.shape}")
    for e in evs:
        if nat.ptr(e.d_scores) % 16 or e.d_bits.data_ptr() % 16:
            raise ParameterError("window buffers must be 16-byte aligned")
    sl = torch.tensor([nat.ptr(evs[i].d_scores) for i in order], dtype=torch.int64, device="cuda")
    bl = torch.tensor([evs[i].d_bits.data_ptr() for i in order], dtype=torch.int64, device="cuda")
    c = th.shape[0]
    acc = torch.empty((len(order), c), dtype=torch.float64, device="cuda")
    sav = torch.empty((len(order), c), dtype=torch.float64, device="cuda")
    nat.check(nat.load_library().ee_eval_thresholds_windows(
        nat.workspace(), sl.data_ptr(), bl.data_ptr(), len(order), e0.n, e0.r, e0.serve.ctypes.data,
        float(e0.vanilla_ms), th.ctypes.data, c, acc.data_ptr(), sav.data_ptr(),
        nat.stream_handle(torch)))
    acc._eeb200_keep = (sl, bl)  # pointer lists live until the stream has used them
    return acc, sav
