#!/usr/bin/env python3
"""Per-stage latency of the packed decode GEMV inside the real decode graph
(EET device trace, CTA 0 of each launch): us since kernel start at
[weights issued, PDL wait passed, X staged, MMA done, reduced, end]."""
import ctypes as C, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402
from paper_2104_12470_b200 import _lib  # noqa: E402

def main():
    b = int(os.environ.get("B", "16"))
    cfg = eet.ModelConfig(b, 1024, 24, 16, 512, 1024, datatype_label="fp16")
    w = eet.random_weights(cfg, 50257, seed=0)
    rng = np.random.default_rng(0)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=512)] for _ in range(b)]
    req = eet.GenerationRequest(prompts=prompts, steps=16)
    pool = eet.BufferPool()
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    _lib.lib().eet_debug_ktrace(1, None, None)
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    out = np.zeros((4096, 8), dtype=np.int64); n = C.c_int()
    _lib.lib().eet_debug_ktrace(0, out.ctypes.data_as(C.c_void_p), C.byref(n))
    recs = out[:n.value]
    for key in sorted(set(map(tuple, recs[:, 6:8]))):
        sel = recs[(recs[:, 6] == key[0]) & (recs[:, 7] == key[1])]
        med = np.median(sel[:, :6], axis=0) / 1e3
        print(f"N{key[0]} K{key[1] % 100000}{' LN' if key[1] >= 100000 else ''} x{len(sel)}: "
              + " ".join(f"{v:.2f}" for v in med))

if __name__ == "__main__":
    main()
