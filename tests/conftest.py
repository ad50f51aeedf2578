"""Shared test fixtures.

``gpu``-marked tests run the CUDA path on a B200 (``pytest -m gpu``); all
other tests run on CPU: the oracle against the golden vectors from the real
reference, host-side plumbing, and that the C-ABI library loads and exports
every symbol ``include/eet_b200.h`` declares.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def golden_meta(data) -> dict:
    import json
    return json.loads(bytes(data["meta"]).decode())


def combined_close(ours, ref, rtol, what=""):
    """North-star tolerance on valid rows: |d| <= rtol*|ref| + rtol*rms(ref)
    (pure rtol is unsatisfiable near zero)."""
    ours = np.asarray(ours, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref * ref))) if ref.size else 0.0
    err = np.abs(ours - ref)
    bound = rtol * np.abs(ref) + rtol * rms
    bad = err > bound
    if bad.any():
        i = np.unravel_index(int(np.argmax(err - bound)), err.shape)
        raise AssertionError(
            f"{what}: {int(bad.sum())}/{bad.size} elements outside rtol {rtol}; "
            f"worst at {i}: ours {ours[i]!r} ref {ref[i]!r} (rms {rms:.3g})")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
