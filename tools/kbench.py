#!/usr/bin/env python3
"""Per-kernel micro-benchmarks at the BASELINE shapes (CUDA events around N
back-to-back launches on one stream). Development tool; bench.py is the
contract.

    python tools/kbench.py [--only gemv,ln,decode,prefill,gemm]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2104_12470_b200 as eet  # noqa: E402
from paper_2104_12470_b200 import _lib  # noqa: E402

HBM = 6548.5
TC = 1659.7


def timeit(fn, n=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3     # us


def gemm_case(dt, M, N, K):
    td = {1: torch.bfloat16, 2: torch.float16, 0: torch.float32}[dt]
    A = torch.randn(M, K, device="cuda").to(td)
    B = torch.randn(N, K, device="cuda").to(td)
    C = torch.empty(M, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def f():
        _lib.call("eet_gemm", dt, A.data_ptr(), B.data_ptr(), None, C.data_ptr(), M, N, K, N, st)
    us = timeit(f)
    es = 4 if dt == 0 else 2
    by = (M * K + N * K) * es + M * N * 4
    fl = 2.0 * M * N * K
    return {"shape": [M, N, K], "us": round(us, 2), "GB/s": round(by / us / 1e3, 1),
            "TFLOP/s": round(fl / us / 1e6, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="gemv,ln,gemm,decode,prefill")
    a = ap.parse_args()
    only = set(a.only.split(","))
    out = {}
    if "gemv" in only:
        for M in (1, 16):
            for N, K in ((3072, 1024), (1024, 1024), (4096, 1024), (1024, 4096), (50257, 1024)):
                out[f"gemv_fp16_M{M}_{N}x{K}"] = gemm_case(2, M, N, K)
    if "gemm" in only:
        for M, N, K in ((8192, 3072, 1024), (15133, 6144, 2048), (15133, 2048, 8192),
                        (32768, 16384, 4096), (2048, 36864, 12288)):
            out[f"gemm_bf16_{M}x{N}x{K}"] = gemm_case(1, M, N, K)
    if "ln" in only:
        for rows, h in ((16, 1024), (8192, 1024), (32768, 4096)):
            x = torch.randn(rows, h, device="cuda")
            g = torch.ones(h, device="cuda")
            b = torch.zeros(h, device="cuda")
            y = torch.empty_like(x)
            st = torch.cuda.current_stream().cuda_stream
            us = timeit(lambda: _lib.call("eet_layer_norm", x.data_ptr(), g.data_ptr(), b.data_ptr(),
                                          y.data_ptr(), rows, h, 0, st))
            out[f"ln_{rows}x{h}"] = {"us": round(us, 2), "GB/s": round(rows * h * 8 / us / 1e3, 1)}
    if "decode" in only or "prefill" in only:
        for name, b, h, heads, s, dt in (("c2_b16", 16, 1024, 16, 512, "fp16"),
                                          ("c3", 32, 2048, 16, 1024, "bf16"),
                                          ("c4", 8, 4096, 32, 4095, "bf16")):
            cfg = eet.ModelConfig(b, h, 1, heads, s, s + 1, datatype_label=dt)
            lw = eet.random_weights(eet.ModelConfig(1, h, 1, heads, 1, 1), 8, 0).layers[0]
            kv, acts = eet.preallocate_caches(cfg)
            pool = eet.BufferPool()
            desc = eet.make_batch([s] * b)
            x = torch.randn(b, s, h, device="cuda")
            _lib.profile_enable(True)
            eet.decoder_layer_forward(x, lw, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
            kv.advance(s)
            x1 = torch.randn(b, 1, h, device="cuda")
            for _ in range(5):
                eet.decoder_layer_forward(x1, lw, kv, desc, eet.Phase.INCREMENTAL, pool, acts, 0)
            summ = _lib.profile_summary()
            _lib.profile_enable(False)
            for k, (n, ms, by, fl) in summ.items():
                out[f"layer_{name}_{k}"] = {"launches": n, "us_per_launch": round(ms / n * 1e3, 2),
                                            "GB/s": round(by / (ms / 1e3) / 1e9, 1),
                                            "TFLOP/s": round(fl / (ms / 1e3) / 1e12, 2)}
    for k, v in out.items():
        print(k, json.dumps(v), flush=True)


if __name__ == "__main__":
    main()
