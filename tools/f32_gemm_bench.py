#!/usr/bin/env python3
"""fp32-mode GEMM at the c1 shapes through eet_gemm: us per call (CUDA
events around 50 back-to-back calls). Run with EET_F32_GEMM=ffma for the
FFMA path (default: 3xTF32 on tcgen05)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2104_12470_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
tag = os.environ.get("EET_F32_GEMM", "tf32x3")
for (M, N, K) in [(205, 2304, 768), (205, 768, 768), (205, 3072, 768), (205, 768, 3072), (2048, 3072, 1024)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    C = torch.empty(M, N, device="cuda")
    call = lambda: _lib.call("eet_gemm", 0, A.data_ptr(), B.data_ptr(), None, C.data_ptr(), M, N, K, N, st)  # noqa: E731
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"{tag} M{M} N{N} K{K}: {us:.1f} us  {2 * M * N * K / us / 1e6:.1f} TFLOP/s", flush=True)
