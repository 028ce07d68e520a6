"""Shared helpers and fixtures.

`make_chain` / `make_record` build the same profiles and records as the
reference's test helpers (pkg/tests/conftest.py:19-42), so fixtures generated
from the reference (tests/golden/) line up with what these tests construct.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2312_05385_b200.graph import ModelProfile  # noqa: E402
from paper_2312_05385_b200.trace import RampSignal, RequestRecord  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")


def make_chain(n, layer_ms=10.0, ramp_ms=0.5, batches=(1,), name="chain", batch_scale=1.0):
    """Linear n-node model; every non-output node carries a ramp cost."""
    nodes = [f"n{i}" for i in range(n)]
    scale = {b: 1.0 + batch_scale * (b - 1) for b in batches}
    lat = {x: {b: layer_ms * scale[b] for b in batches} for x in nodes}
    ramp = {x: {b: ramp_ms * scale[b] for b in batches} for x in nodes[:-1]}
    edges = list(zip(nodes, nodes[1:]))
    return ModelProfile(nodes, edges, lat, ramp, nodes[-1], name=name)


def make_record(rid, arrival, signals, final):
    return RequestRecord(rid, arrival, {s: RampSignal(e, l) for s, (e, l) in signals.items()}, final)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def kernels_random():
    data = np.load(os.path.join(GOLDEN, "kernels_random.npz"))
    out = []
    for w in range(10):
        out.append({k: data[f"w{w}_{k}"] for k in
                    ("scores", "cext", "serve", "vanilla", "th", "acc", "sav", "acc_numpy",
                     "sav_numpy", "sites")})
    return out


@pytest.fixture(scope="session")
def cuda():
    """The GPU tests never skip: no device means the run is broken, not partial."""
    import torch

    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    from paper_2312_05385_b200 import _native

    _native.load_library()
    return torch
