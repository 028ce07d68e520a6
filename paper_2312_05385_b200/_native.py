"""ctypes binding of libeeb200.so (C ABI: include/eeb200.h).

There is exactly one implementation behind this module — the sm_100a kernels.
If the shared library is missing, or no CUDA device is visible, every entry
point raises; nothing falls back to a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading

from paper_2312_05385_b200.errors import NativeError, ParameterError

LIB_NAME = "libeeb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

EE_OK = 0
EE_ERR_ARG = -1
EE_ERR_CUDA = -2
EE_ERR_NOT_BINARY = -3
EE_ERR_RAMPS = -4

MODE_AUTO = 0
MODE_EXACT = 1
MODE_HIST = 2
MODE_FLAG_RESIDENT = 0x100  # EE_MODE_FLAG_RESIDENT: immutable resident window
MODES = {"auto": MODE_AUTO, "exact": MODE_EXACT, "hist": MODE_HIST}
EXACT_N_MAX = 4096
TUNE_N_MAX = 65536
MAX_RAMPS = 31

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/eeb200.h one to one.
SIGNATURES = {
    "ee_version": (ctypes.c_char_p, []),
    "ee_last_error": (ctypes.c_char_p, []),
    "ee_device_sm_count": (ctypes.c_int, [ctypes.POINTER(_c_i32)]),
    "ee_workspace_create": (ctypes.c_int, [ctypes.POINTER(_vp)]),
    "ee_workspace_destroy": (ctypes.c_int, [_vp]),
    "ee_exit_sites": (ctypes.c_int, [_vp, _c_i64, _c_i32, _vp, _vp, _vp]),
    "ee_pack_correct": (ctypes.c_int, [_vp, _c_i64, _c_i32, _vp, _vp, _vp]),
    "ee_decision_scores": (ctypes.c_int, [_vp, _c_i64, _c_i32, _c_i32, _vp, _vp]),
    "ee_eval_thresholds": (
        ctypes.c_int,
        [_vp, _vp, _vp, _c_i64, _c_i32, _vp, ctypes.c_double, _vp, _c_i64, _c_i32,
         _vp, _vp, _vp, _vp, _vp],
    ),
    "ee_synth_columns": (
        ctypes.c_int,
        [_vp, _c_i64, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _vp, _c_i32, _vp, _vp, _c_i32,
         ctypes.c_double, ctypes.c_double, ctypes.c_double, _c_i32, _vp, _vp, _vp],
    ),
    "ee_finalize_hist": (
        ctypes.c_int,
        [_vp, _vp, _vp, _c_i64, _c_i32, _c_i64, _vp, ctypes.c_double, _vp, _vp, _vp],
    ),
    "ee_profile_enable": (ctypes.c_int, [_vp, _c_i32]),
    "ee_workspace_set_special": (ctypes.c_int, [_vp, _c_i32]),
    "ee_workspace_set_diag_version": (ctypes.c_int, [_vp, _c_i32]),
    "ee_gemm_bf16": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _c_i32, _c_i64, _c_i64, _c_i64, _c_i32, _vp]),
    "ee_eval_thresholds_host": (ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i32, _vp, ctypes.c_double,
                                                _vp, _c_i64, _c_i32, _vp, _vp, _c_i32, _vp]),
    "ee_eval_counts_host": (ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i32, _vp, _c_i64, _vp, _vp, _c_i32, _vp]),
    "ee_pack_correct_host": (ctypes.c_int, [_vp, _c_i64, _c_i32, _vp, _c_i32]),
    "ee_diag_trace": (ctypes.c_int, [_vp, _vp]),
    "ee_tune_profile": (ctypes.c_int, [_vp, _vp]),
    "ee_l2_flush": (ctypes.c_int, [_vp, _c_i64, _vp]),
    "ee_profile_read": (ctypes.c_int, [_vp, ctypes.c_char_p, _c_i64]),
    "ee_tune": (
        ctypes.c_int,
        [_vp, _vp, _vp, _c_i64, _c_i32, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
         ctypes.c_double, _c_i32, _vp, _vp, _vp, _c_i32, _vp],
    ),
    "ee_exit_controller": (
        ctypes.c_int,
        [_vp, _vp, _c_i32, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _c_i32, _vp, _c_i32, _c_i32,
         ctypes.c_double, _vp, _vp, _vp, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "ee_exit_from_logits": (
        ctypes.c_int,
        [_vp, _vp, _c_i64, _c_i32, _c_i32, ctypes.c_double, _vp, _vp, _vp, _c_i32, _vp, _vp, _vp,
         _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "ee_compact_rows": (ctypes.c_int, [_vp, _c_i64, _vp, _vp, _c_i64, _vp, _vp]),
    "ee_conv_bf16": (ctypes.c_int, [_vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _c_i32, _c_i32,
                                    _c_i32, _c_i32, _c_i32, _vp, _vp, _c_i32, _vp, _vp, _c_i64, _vp]),
    "ee_conv_workspace_size": (_c_i64, [_c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32,
                                        _c_i32]),
    "ee_sequential_sum": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _vp]),
    "ee_defer_plan": (ctypes.c_int, [_vp, _c_i32, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _c_i32, _vp]),
    "ee_defer_finish": (ctypes.c_int, [_vp, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _c_i32,
                                       _vp]),
    "ee_im2col_bf16": (ctypes.c_int, [_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32,
                                      _c_i32, _c_i32, _vp, _vp]),
    "ee_maxpool_nhwc_bf16": (ctypes.c_int, [_vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32,
                                            _vp, _vp]),
    "ee_bias_act_bf16": (ctypes.c_int, [_vp, _vp, _vp, _c_i32, _c_i64, _c_i32, _vp, _vp]),
    "ee_seg_chain_create": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _vp, _vp, _vp]),
    "ee_seg_chain_launch": (ctypes.c_int, [_vp, _vp]),
    "ee_seg_chain_destroy": (None, [_vp]),
    "ee_scatter_signals": (ctypes.c_int, [_vp, _vp, _vp, _c_i64, _vp, _vp, _vp]),
    "ee_compact_fill": (ctypes.c_int, [_vp, _c_i64, _vp, _vp, _c_i64, _vp, _c_i32, _vp, _vp, _vp, _vp]),
    "ee_compact_meta": (ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i32, _vp, _vp, _vp, _vp]),
    "ee_gemm_bf16_tn": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _vp]),
    "ee_gemm_bf16_ex": (
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp,
         _c_i64, _vp],
    ),
    "ee_gemm_bf16_res": (
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _vp,
         _c_i64, _vp],
    ),
    "ee_gemm_workspace_size": (_c_i64, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_i32]),
    "ee_pool_bf16": (ctypes.c_int, [_vp, _c_i32, _c_i64, _c_i32, _c_i32, _vp, _vp]),
    "ee_pool_nhwc_bf16": (ctypes.c_int, [_vp, _c_i32, _c_i64, _c_i32, _c_i32, _vp, _vp]),
    "ee_classify_candidates": (ctypes.c_int, [_vp, _c_i64, _c_i32, _vp, _vp, _vp]),
    "ee_kv_append_bf16": (ctypes.c_int, [_vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i64, _vp, _vp]),
    "ee_add_layernorm_bf16": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_double, _c_i64, _c_i32, _vp, _vp]),
    "ee_windows_counts": (ctypes.c_int, [_vp, _vp, _vp, _c_i32, _c_i64, _c_i32, _vp, _c_i64, _vp, _vp]),
    "ee_windows_finalize": (ctypes.c_int, [_vp, _vp, _c_i32, _c_i64, _c_i32, _vp, ctypes.c_double, _vp,
                                           _c_i64, _vp, _vp, _vp]),
    "ee_eval_thresholds_windows": (ctypes.c_int, [_vp, _vp, _vp, _c_i32, _c_i64, _c_i32, _vp, ctypes.c_double,
                                                  _vp, _c_i64, _vp, _vp, _vp]),
    "ee_decode_attention_bf16": (ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _c_i64, _vp, _vp]),
    "ee_eval_lattice": (
        ctypes.c_int,
        [_vp, _vp, _vp, _c_i64, _c_i32, _vp, ctypes.c_double, _vp, _c_i32, _vp, _vp, _vp],
    ),
}

_lib = None
_lock = threading.Lock()
_tls = threading.local()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the shared library (no CUDA call is made here)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == EE_OK:
        return
    msg = load_library().ee_last_error().decode(errors="replace")
    if rc in (EE_ERR_ARG, EE_ERR_RAMPS):
        raise ParameterError(msg)
    if rc == EE_ERR_NOT_BINARY:
        raise ValueError(msg)
    raise NativeError(f"eeb200 error {rc}: {msg}")


def torch_cuda():
    """Return torch with a usable CUDA device, or raise (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeError("eeb200 needs a CUDA device (sm_100a); none is visible and there is no CPU fallback")
    return torch


class _Workspace:
    def __init__(self):
        lib = load_library()
        h = _vp()
        check(lib.ee_workspace_create(ctypes.byref(h)))
        self.handle = h
        if os.environ.get("EEB200_DIAG_VERSION"):  # A/B runs of the diagonal kernels
            check(lib.ee_workspace_set_diag_version(h, int(os.environ["EEB200_DIAG_VERSION"])))

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            if _lib is not None and self.handle:
                _lib.ee_workspace_destroy(self.handle)
        except Exception:
            pass


def workspace() -> ctypes.c_void_p:
    """Per-thread workspace handle (device scratch + pinned staging)."""
    ws = getattr(_tls, "ws", None)
    if ws is None:
        ws = _Workspace()
        _tls.ws = ws
    return ws.handle


def set_diag_version(version: int = 4) -> None:
    """4 = k_diag3 where it applies, else k_diag2 (default); 2 = k_diag2 where it
    applies; 1 = the first diagonal kernel only."""
    check(load_library().ee_workspace_set_diag_version(workspace(), int(version)))


def set_special(on: bool = True) -> None:
    """Enable/disable family-specialised sweeps on this thread's workspace."""
    check(load_library().ee_workspace_set_special(workspace(), int(on)))


def profile_enable(on: bool = True) -> None:
    check(load_library().ee_profile_enable(workspace(), int(on)))


def profile_read() -> dict:
    """{kernel: {"launches": L, "ms": T}} since the last read (synchronises)."""
    import json

    buf = ctypes.create_string_buffer(1 << 16)
    check(load_library().ee_profile_read(workspace(), buf, len(buf)))
    return json.loads(buf.value.decode())


def l2_flush(buf) -> None:
    """Evict L2 by streaming over `buf` (a CUDA tensor larger than L2), same carveout as the sweeps."""
    import torch

    check(load_library().ee_l2_flush(buf.data_ptr(), buf.numel() * buf.element_size(),
                                     stream_handle(torch)))


def stream_handle(torch) -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return t.data_ptr() if t is not None and t.numel() > 0 else 0
