"""The reference's own tests, re-run with the B200 kernels swapped into
`eesim._kernels` (tools/run_reference_suite.py)."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "eesim")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.isdir(REF) and os.path.isdir(REF_TESTS)),
                    reason="reference not installed under baseline/_ref (build-container artifact)")
def test_reference_engine_tuner_kernel_suites_pass_on_gpu(cuda):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "run_reference_suite.py"),
                          "test_kernels.py", "test_engine.py", "test_tuner.py", "test_ramps.py"],
                         capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
