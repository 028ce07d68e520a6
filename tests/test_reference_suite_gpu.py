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


@pytest.mark.gpu
@pytest.mark.skipif(not (os.path.isdir(REF) and os.path.isdir(REF_TESTS)),
                    reason="reference not installed under baseline/_ref (build-container artifact)")
def test_reference_acceptance_and_serving_suites_pass_on_gpu(cuda):
    """The reference's acceptance criteria c2-c4 (pkg/tests/test_acceptance.py:88-148:
    hill-climb near-optimality vs the grid oracle, tuner speed, 1000-case
    monotonicity) and its serving-loop tests, with every WindowEvaluator
    evaluating on the B200 (tune, grid_oracle, the serving loop's adaptation)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "run_reference_suite.py"),
                          "test_acceptance.py", "test_serving.py"],
                         capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-4000:] + out.stderr[-2000:]
    report = os.environ.get("EEB200_PARITY_REPORT")
    if report:
        with open(report + ".acceptance.txt", "w") as fh:
            fh.write(out.stdout + out.stderr)
    print(tail)
    assert out.returncode == 0, tail
