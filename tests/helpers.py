"""Test-only helpers shared by several test modules."""

from __future__ import annotations

import hashlib
import json

import numpy as np


def digest_records(records) -> str:
    """Same digest as tests/golden/make_golden.py."""
    h = hashlib.sha256()
    for rec in records:
        obj = {"id": rec.id, "a": rec.arrival_ms, "f": rec.final_label,
               "s": {k: [v.err.hex(), v.label] for k, v in sorted(rec.ramp_signals.items())}}
        h.update(json.dumps(obj, sort_keys=True).encode())
    return h.hexdigest()


def config4_profile():
    from conftest import make_chain

    return make_chain(13, layer_ms=1.0, ramp_ms=0.01)


def config4_curve(sites):
    return {x.position: 0.5 + (0.95 - 0.5) * i / 11 for i, x in enumerate(sites)}


def diagonal(c=64, r=12):
    return np.repeat((np.arange(c) / (c - 1.0))[:, None], r, axis=1)


def axis_sweep(r=12, m=64, base=0.3):
    th = np.full((r * m, r), base)
    for j in range(r):
        th[j * m:(j + 1) * m, j] = np.arange(m) / (m - 1.0)
    return th
