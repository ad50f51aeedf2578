#!/usr/bin/env python3
"""Decode GEMV chain in a CUDA graph with HBM-cold weights: 24 layers x
[QKV 3072x1024, O 1024x1024, W1 4096x1024, W2 1024x4096] with distinct
weights per layer (604 MB, like the c2 decode step), packed path vs tcgen05
path; prints per-launch averages. Development tool."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2104_12470_b200 import _lib  # noqa: E402

def main():
    M = int(os.environ.get("M", "16"))
    shapes = [(3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096)]
    Ws = [[(torch.randn(N, K, device="cuda") * 0.02).half() for N, K in shapes] for _ in range(24)]
    Xs = {K: torch.randn(M, K, device="cuda").half() for _, K in shapes}
    out = torch.empty(M, 4096, device="cuda")
    st = lambda: torch.cuda.current_stream().cuda_stream
    for l in range(24):
        for (N, K), W in zip(shapes, Ws[l]):
            if K == 1024:
                _lib.call("eet_gemv_packed", 2, W.data_ptr(), N, K, Xs[K].data_ptr(), M, out.data_ptr(), 1, st())
    torch.cuda.synchronize()
    def chain(packed, which):
        for l in range(24):
            for i, ((N, K), W) in enumerate(zip(shapes, Ws[l])):
                if i not in which:
                    continue
                if packed and K == 1024:
                    _lib.call("eet_gemv_packed", 2, W.data_ptr(), N, K, Xs[K].data_ptr(), M, out.data_ptr(), 0, st())
                else:
                    _lib.call("eet_gemm", 2, Xs[K].data_ptr(), W.data_ptr(), None, out.data_ptr(), M, N, K, N, st())
    for packed in (True, False):
        for which, name in (((0, 1, 2, 3), "all4"), ((0,), "qkv"), ((2,), "w1"), ((3,), "w2"), ((1,), "o")):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                chain(packed, which); torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    chain(packed, which)
                g.replay(); torch.cuda.synchronize()
                best = 1e9
                for _ in range(5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s); g.replay(); b.record(s); torch.cuda.synchronize()
                    best = min(best, a.elapsed_time(b))
            n = 24 * len(which)
            byts = sum(shapes[i][0] * shapes[i][1] * 2 for i in which) * 24
            print(f"M{M} {'packed' if packed else 'tcgen05'} {name}: {best * 1e3 / n:.2f} us/launch, "
                  f"{byts / (best * 1e-3) / 1e12:.2f} TB/s", flush=True)

if __name__ == "__main__":
    main()
