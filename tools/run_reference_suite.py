"""Run the REFERENCE's own test files with the B200 kernels installed into
`eesim._kernels` (the drop-in seam).

Needs the reference installed under baseline/_ref (pip --target, git-ignored)
and its tests copied to baseline/_ref_tests. Every WindowEvaluator in the
reference — tune, grid_oracle, evaluate_window, estimate_utilities, the
serving loop's adaptation — then evaluates on the GPU.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(1, ROOT)

import eesim._kernels  # noqa: E402

from paper_2312_05385_b200 import kernels  # noqa: E402

kernels.install_into(eesim._kernels)
assert getattr(eesim._kernels.eval_thresholds, "__wrapped__", None) is kernels.eval_thresholds

import pytest  # noqa: E402

files = sys.argv[1:] or ["test_kernels.py", "test_engine.py", "test_tuner.py", "test_ramps.py",
                         "test_serving.py", "test_acceptance.py"]
tests = os.path.join(ROOT, "baseline", "_ref_tests")
args = [os.path.join(tests, f) if f.endswith(".py") else f for f in files]
sys.exit(pytest.main(args + ["-q", "-p", "no:cacheprovider", "--rootdir", tests, "-rA"]))
