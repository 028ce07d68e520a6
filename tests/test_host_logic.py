"""Host-side logic of the B200 paths that needs no GPU: compaction segments and
buckets, the device decode-schedule state layout shared with the C ABI, and
the GEMM planner's workspace query (the library loads and plans without a
device)."""

from __future__ import annotations

import ctypes

import pytest

from paper_2312_05385_b200 import _native
from paper_2312_05385_b200.ee_infer import compaction_buckets, compaction_segments


def test_compaction_segments_end_at_ramps_and_the_classifier():
    assert compaction_segments([0, 2, 3, 5, 6, 8], 10) == [(0, 0), (1, 2), (3, 3), (4, 5), (6, 6),
                                                          (7, 8), (9, 9)]
    assert compaction_segments(list(range(16)), 17) == [(j, j) for j in range(17)]
    assert compaction_segments([], 3) == [(0, 2)]


@pytest.mark.parametrize("b", [1, 7, 32, 48, 64, 256, 300])
def test_compaction_buckets_cover_every_live_count(b):
    bk = compaction_buckets(b)
    assert bk[-1] == b and bk == sorted(set(bk))
    granule = max(1, b // 16)
    for n in range(1, b + 1):
        best = min(x for x in bk if x >= n)
        assert best - n < max(granule, n)  # never more than one granule (or 2x below it) of padding
    assert len(bk) <= 17 + granule.bit_length() + 1  # 16 multiples, B itself, powers of two


def test_defer_state_layout_matches_the_c_struct():
    """ee_defer_state (include/eeb200.h): 13 pointers + n_max + padding = 112 bytes,
    the ctypes mirror generative.py builds must have the same size and order."""
    fields = ["step", "n_def", "qpos", "def_step", "mem_cnt", "spos", "h_exit", "h_err", "h_lab",
              "h_final", "h_cnt", "h_kind", "h_qbase"]

    class State(ctypes.Structure):
        _fields_ = [(k, ctypes.c_void_p) for k in fields] + [("n_max", ctypes.c_int32),
                                                              ("pad_", ctypes.c_int32)]

    assert ctypes.sizeof(State) == 112
    assert State.n_max.offset == 13 * 8
    import inspect

    from paper_2312_05385_b200 import generative

    src = inspect.getsource(generative.TokenEEDecoder._device_state)
    for k in fields:
        assert f'"{k}"' in src


def test_gemm_planner_without_a_device():
    lib = _native.load_library()
    # M = 32 decode GEMM, auto split-K: a positive fp32 partial workspace
    w = lib.ee_gemm_workspace_size(32, 1024, 4096, 0, 0, 1)
    assert w > 0
    # unsplit swap kernel and the pair kernel need none
    assert lib.ee_gemm_workspace_size(32, 1024, 4096, 1, 0, 1) == 0
    assert lib.ee_gemm_workspace_size(8192, 2304, 768, 0, 0, 1) == 0
    # bad shapes / paths are rejected
    assert lib.ee_gemm_workspace_size(0, 1, 1, 0, 0, 1) < 0
    assert lib.ee_gemm_workspace_size(32, 32, 64, 0, 9, 1) < 0
