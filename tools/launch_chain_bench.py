#!/usr/bin/env python3
"""Per-link cost of a chain of dependent (nearly) empty kernels captured in a
CUDA graph, with / without programmatic dependent launch. Development tool."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2104_12470_b200 import _lib  # noqa: E402

def main():
    n = 200
    for ctas in (1, 148, 296):
        for pdl in (0, 1):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                f = lambda: _lib.call("eet_debug_launch_chain", n, ctas, pdl, None, s.cuda_stream)
                f(); torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    f()
                g.replay(); torch.cuda.synchronize()
                best = 1e9
                for _ in range(5):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s); g.replay(); b.record(s); torch.cuda.synchronize()
                    best = min(best, a.elapsed_time(b))
            print(f"ctas {ctas} pdl {pdl}: {best * 1e3 / n:.2f} us per link", flush=True)

if __name__ == "__main__":
    main()
