#!/usr/bin/env python3
"""Phase timeline of the fused decode kernels inside the real c2 decode graph
(eet_debug_aotrace): for the last traced launches of attn_o.cu or
qkv_attn_o.cu, per-CTA phase durations (us) and the launch span."""
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
    req = eet.GenerationRequest(prompts=prompts, steps=6)
    pool = eet.BufferPool()
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    _lib.lib().eet_debug_aotrace(1, None, None)
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    out = np.zeros((8192, 8), dtype=np.int64); n = (C.c_int * 2)()
    _lib.lib().eet_debug_aotrace(0, out.ctypes.data_as(C.c_void_p), n)
    per = b * 16
    if n[1]:                                   # qkv_attn_o: [id, start, wait, ln, qkv, attn, gather, end]
        r = out[4096:4096 + n[1]]
        r = r[np.argsort(r[:, 1])]
        names = ["wait-start", "LN", "QKV", "attn", "gather", "tail"]
        launches = [r[i:i + per] for i in range(0, len(r) - per + 1, per)]
        print(f"qkv_attn_o: {len(launches)} launches of {per} CTAs; phase median/max (us)")
        print("  span   " + "  ".join(f"{x:>11s}" for x in names))
        for L in launches[-6:]:
            t0 = L[:, 1].min()
            ph = np.diff(L[:, 1:8], axis=1) / 1e3
            print(f"  {(L[:, 7].max() - t0) / 1e3:6.2f} " + "  ".join(
                f"{m:5.2f}/{x:5.2f}" for m, x in zip(np.median(ph, 0), ph.max(0))) +
                f"  wait spread {(L[:, 2].max() - L[:, 2].min()) / 1e3:5.2f}")
    if n[0]:
        r = out[:n[0]]
        r = r[np.argsort(r[:, 2])]
        launches = [r[i:i + per] for i in range(0, len(r) - per + 1, per)]
        print(f"attn_o: {len(launches)} launches of {per} CTAs; phases per CTA (us): median / max")
        print("launch  span  start-spread  wait-start  attn  gather  tail")
        for L in launches[-8:]:
            t0 = L[:, 2].min()
            span = (L[:, 6].max() - t0) / 1e3
            ph = np.stack([(L[:, 3] - L[:, 2]), (L[:, 4] - L[:, 3]), (L[:, 5] - L[:, 4]), (L[:, 6] - L[:, 5])], 1) / 1e3
            med, mx = np.median(ph, 0), ph.max(0)
            print(f"  {span:6.2f}  {(L[:, 2].max() - t0) / 1e3:6.2f}  " +
                  "  ".join(f"{a:5.2f}/{m:5.2f}" for a, m in zip(med, mx)) +
                  f"   wait-passed spread {(L[:, 3].max() - L[:, 3].min()) / 1e3:5.2f}")


if __name__ == "__main__":
    main()
