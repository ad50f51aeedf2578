#!/usr/bin/env python3
"""Decode-GEMV micro-benchmark: per-launch time of back-to-back launches
captured in a CUDA graph (the way generate runs them), old tcgen05 split-K
path (eet_gemm, M <= 32) vs the packed mma.sync path (eet_gemv_packed).
Development tool."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2104_12470_b200 import _lib  # noqa: E402

def graph_time(fn, n=50, reps=5):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
        g.replay(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / n * 1e3)
    return best

def main():
    M = int(os.environ.get("M", "16"))
    for N, K in ((3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096), (50257, 1024)):
        W = (torch.randn(N, K, device="cuda") * 0.02).half()
        X = torch.randn(M, K, device="cuda").half()
        out = torch.empty(M, N, device="cuda")
        ref = X.float() @ W.float().t()
        st = lambda: torch.cuda.current_stream().cuda_stream
        _lib.call("eet_gemv_packed", 2, W.data_ptr(), N, K, X.data_ptr(), M, out.data_ptr(), 1, st())
        torch.cuda.synchronize()
        err = (out - ref).abs().max().item()
        t_new = graph_time(lambda: _lib.call("eet_gemv_packed", 2, W.data_ptr(), N, K, X.data_ptr(), M,
                                             out.data_ptr(), 0, torch.cuda.current_stream().cuda_stream))
        t_old = graph_time(lambda: _lib.call("eet_gemm", 2, X.data_ptr(), W.data_ptr(), None, out.data_ptr(),
                                             M, N, K, N, torch.cuda.current_stream().cuda_stream))
        mb = N * K * 2 / 1e6
        print(f"N{N} K{K} M{M}: packed {t_new:.2f} us ({mb / t_new * 1e-3 * 1e3:.0f} GB/s)  "
              f"tcgen05 {t_old:.2f} us ({mb / t_old * 1e-3 * 1e3:.0f} GB/s)  max|err| {err:.2e}", flush=True)

if __name__ == "__main__":
    main()
