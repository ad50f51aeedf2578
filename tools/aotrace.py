#!/usr/bin/env python3
"""Phase timeline of the fused decode attention + out-projection (attn_o.cu)
inside the real c2 decode graph (eet_debug_aotrace): for the last traced
launches, per-CTA phase durations (us) and the launch span."""
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
    out = np.zeros((4096, 8), dtype=np.int64); n = C.c_int()
    _lib.lib().eet_debug_aotrace(0, out.ctypes.data_as(C.c_void_p), C.byref(n))
    r = out[:n.value]
    r = r[np.argsort(r[:, 2])]
    per = b * 16
    launches = [r[i:i + per] for i in range(0, len(r) - per + 1, per)]
    print(f"{len(launches)} launches of {per} CTAs; phases per CTA (us): median / max")
    print("launch  span  start-spread  wait-start  attn  gather  tail  (end - first start)")
    for L in launches[-8:]:
        t0 = L[:, 2].min()
        span = (L[:, 6].max() - t0) / 1e3
        ph = np.stack([(L[:, 3] - L[:, 2]), (L[:, 4] - L[:, 3]), (L[:, 5] - L[:, 4]), (L[:, 6] - L[:, 5])], 1) / 1e3
        med, mx = np.median(ph, 0), ph.max(0)
        print(f"  {span:6.2f}  {(L[:, 2].max() - t0) / 1e3:6.2f}  " +
              "  ".join(f"{a:5.2f}/{m:5.2f}" for a, m in zip(med, mx)) +
              f"   wait-passed spread {(L[:, 3].max() - L[:, 3].min()) / 1e3:5.2f}  attn-done spread "
              f"{(L[:, 4].max() - L[:, 4].min()) / 1e3:5.2f}")


if __name__ == "__main__":
    main()
