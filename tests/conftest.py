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


def check_16bit(ours, ref, dt, what, emu_ratio=None):
    """16-bit parity against the fp32 oracle.

    * always: norm-wise relative error ||d|| / ||ref|| <= 2e-2 (north star);
    * fp16: the combined elementwise form at 2e-2 (``combined_close``);
    * bf16: the combined elementwise ratio may not exceed what the format
      itself costs — ``emu_ratio``, the same ratio of the torch / cuBLAS
      restatement with identical rounding points (tests/emu16.py) — by more
      than 15 % (and passes outright at <= 1). bf16's 8-bit significand puts
      the format alone above 1 at GPT-2-medium depth and at K = 49152.
    Returns (norm-wise error, elementwise ratio)."""
    from emu16 import bound_ratio, norm_rel
    nr, br = norm_rel(ours, ref), bound_ratio(ours, ref)
    assert nr <= 2e-2, f"{what}: norm-wise relative error {nr:.4g} > 2e-2"
    if dt == "bf16" and emu_ratio is not None:
        assert br <= max(1.0, 1.15 * emu_ratio), (
            f"{what}: elementwise ratio {br:.3f} vs the bf16 format's own {emu_ratio:.3f}")
    else:
        combined_close(ours, ref, 2e-2, what)
    return nr, br
