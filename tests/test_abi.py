"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/eeb200.h declares (no compute calls here)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2312_05385_b200 import _native, kernels
from paper_2312_05385_b200.errors import ParameterError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "eeb200.h")).read()
    return sorted(set(re.findall(r"\b(ee_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("ee_exit_sites", "ee_eval_thresholds", "ee_eval_lattice", "ee_pack_correct",
                 "ee_decision_scores", "ee_workspace_create", "ee_workspace_destroy"):
        assert name in syms


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    for name in header_symbols():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_native.SIGNATURES) == set(header_symbols())


def test_version_string_without_gpu():
    lib = _native.load_library()
    assert b"sm_100a" in lib.ee_version()


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_shape_errors_are_raised_before_any_device_work():
    import numpy as np

    s = np.zeros((3, 2))
    with pytest.raises(ParameterError):
        kernels.exit_sites(s, np.zeros(3))
    with pytest.raises(ParameterError):
        kernels.eval_thresholds(s, np.ones((3, 2)), np.ones(3), 1.0, np.zeros((2, 2)))
    with pytest.raises(ParameterError):
        kernels.eval_thresholds(s, np.ones((3, 3)), np.ones(2), 1.0, np.zeros((2, 2)))
    with pytest.raises(ParameterError):
        kernels.eval_thresholds(s, np.ones((3, 3)), np.ones(3), 1.0, np.zeros((2, 3)))


def test_buffer_errors_follow_cython_memoryview_types():
    import numpy as np

    with pytest.raises(ValueError, match="dtype mismatch"):
        kernels.exit_sites(np.zeros((3, 2), dtype=np.int64), np.zeros(2))
    with pytest.raises(ValueError, match="C-contiguous"):
        kernels.exit_sites(np.zeros((3, 4))[:, ::2], np.zeros(2))
    with pytest.raises(ValueError, match="dimensions"):
        kernels.exit_sites(np.zeros(3), np.zeros(2))
    with pytest.raises(TypeError):
        kernels.exit_sites([[0.1, 0.2]], np.zeros(2))
    with pytest.raises(TypeError):
        kernels.exit_sites(np.zeros((3, 2)), [0.1, 0.2])


def test_backend_surface_mirrors_reference_seam():
    assert kernels.BACKEND == "cuda"
    assert kernels.available_backends() == ["cuda"]
    assert kernels.get_backend("cuda") is kernels
    with pytest.raises(ValueError):
        kernels.get_backend("python")  # no CPU fallback exists

    class Seam:
        pass

    seam = Seam()
    kernels.install_into(seam)
    assert seam.eval_thresholds is kernels.eval_thresholds
    assert seam.exit_sites is kernels.exit_sites


def test_install_into_reference_raises_reference_error_classes():
    """Installed into the reference's `eesim._kernels`, shape errors surface as
    eesim.errors.ParameterError, so `except EESimError` in a
    reference caller still catches them. The checks run before any device work."""
    import importlib
    import sys
    import numpy as np

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "eesim")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, ref)
    try:
        ek = importlib.import_module("eesim._kernels")
        ee = importlib.import_module("eesim.errors")
        saved = (ek.eval_thresholds, ek.exit_sites, ek.BACKEND)
        try:
            kernels.install_into(ek)
            assert ek.BACKEND == "cuda"
            assert ek.eval_thresholds.__wrapped__ is kernels.eval_thresholds
            with pytest.raises(ee.ParameterError, match="columns"):
                ek.eval_thresholds(np.zeros((4, 3)), np.ones((4, 4)), np.zeros(4), 1.0,
                                   np.zeros((2, 2)))
            with pytest.raises(ee.EESimError):
                ek.exit_sites(np.zeros((4, 3)), np.zeros(2))
            with pytest.raises(ValueError, match="dtype"):  # buffer errors keep Cython's types
                ek.exit_sites(np.zeros((4, 3), dtype=np.float32), np.zeros(3))
        finally:
            ek.eval_thresholds, ek.exit_sites, ek.BACKEND = saved
    finally:
        sys.path.remove(ref)


def test_no_gpu_means_loud_failure(monkeypatch):
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(Exception, match="CUDA device"):
        kernels.exit_sites(np.zeros((3, 2)), np.zeros(2))


def test_host_pack_correct_matches_numpy_and_rejects_non_binary():
    """ee_pack_correct_host (the CPU half of ee_eval_thresholds_host) is plain
    host code: bit j of row i = correct_ext[i, j], multi-threaded, exact."""
    from paper_2312_05385_b200 import kernels

    rng = np.random.default_rng(5)
    for n, r1 in [(0, 3), (1, 1), (37, 13), (100_003, 13), (5000, 32)]:
        cext = rng.integers(0, 2, size=(n, r1)).astype(np.float64)
        want = (cext.astype(np.uint64) << np.arange(r1, dtype=np.uint64)).sum(axis=1).astype(np.uint32) \
            if n else np.empty(0, dtype=np.uint32)
        for threads in (1, 3, 0):
            got = kernels.pack_correct_host(cext, n_threads=threads)
            assert np.array_equal(got, want)
    bad = np.zeros((9000, 4))
    bad[7777, 2] = 0.5
    with pytest.raises(ValueError):
        kernels.pack_correct_host(bad)
    bad[7777, 2] = np.nan
    with pytest.raises(ValueError):
        kernels.pack_correct_host(bad)


def test_candidate_family_classification_on_the_host():
    """ee_classify_candidates (host only) sees the families the sweep dispatch
    specialises: diagonal rows, a base vector with one swept ramp (SURVEY 8d's
    C = 768 axis family, NaN base entries and rows equal to the base included),
    and everything else as generic."""
    r = 12
    diag = np.repeat((np.arange(64) / 63.0)[:, None], r, axis=1)
    assert kernels.classify_candidates(diag) == ("diagonal", 64, None)
    diag_nan = np.vstack([diag, np.full((1, r), np.nan)])
    assert kernels.classify_candidates(diag_nan)[:2] == ("diagonal", 64)
    axis = np.full((768, r), 0.3)
    for j in range(r):
        axis[j * 64:(j + 1) * 64, j] = np.arange(64) / 63.0
    kind, m, base = kernels.classify_candidates(axis)
    assert kind == "axis" and m == 64 and np.array_equal(base, np.full(r, 0.3))
    axis2 = axis.copy()
    axis2[:, 5] = np.where(np.arange(768) // 64 == 5, axis2[:, 5], np.nan)  # NaN base entry
    axis2 = np.vstack([axis2, axis2[0:1] * 0 + np.where(np.arange(r) == 5, np.nan, 0.3)])
    kind, m, base = kernels.classify_candidates(axis2)
    assert kind == "axis" and np.isnan(base[5]) and base[0] == 0.3
    rnd = (np.arange(64) / 63.0)[np.random.default_rng(1).integers(0, 64, size=(64, r))]
    assert kernels.classify_candidates(rnd) == ("generic", 0, None)
    two = np.full((4, r), 0.3)
    two[1, 0] = two[1, 1] = 0.9  # two columns changed in one row
    assert kernels.classify_candidates(two)[0] == "generic"
    assert kernels.classify_candidates(np.empty((0, r)))[0] == "generic"


def test_windows_batch_rejects_non_diagonal_rows_before_device_work():
    """ee_eval_thresholds_windows validates its envelope on the host first: a
    non-diagonal candidate matrix (or odd R, or C > 512) is a ParameterError with
    no device call (the fake device pointers below are never dereferenced)."""
    lib = _native.load_library()
    ws = ctypes.c_void_p(1)  # never used before validation fails
    serve = np.zeros(13)
    fake = ctypes.c_void_p(16)
    rnd = np.random.default_rng(0).random((8, 12))
    for th, r in ((rnd, 12), (np.zeros((8, 5)), 5), (np.zeros((600, 12)), 12)):
        th = np.ascontiguousarray(th)
        rc = lib.ee_eval_thresholds_windows(ws, fake, fake, 2, 1000, r, serve.ctypes.data, 10.0,
                                            th.ctypes.data, th.shape[0], fake, fake, None)
        with pytest.raises(ParameterError):
            _native.check(rc)
