#!/usr/bin/env python3
"""Calibration: us per grid-wide barrier (eet_debug_grid_barrier) vs the
PDL link of a CUDA graph (eet_debug_launch_chain)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2104_12470_b200 import _lib  # noqa: E402

for mode in (0, 1):
    for ctas in (144, 148 if mode == 0 else 144):
        v = C.c_float()
        _lib.call("eet_debug_grid_barrier", 2000, ctas, mode, C.byref(v))
        print(f"mode {'flat' if mode == 0 else 'cluster'} ctas {ctas}: {v.value:.3f} us / barrier", flush=True)
