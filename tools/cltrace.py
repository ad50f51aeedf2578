#!/usr/bin/env python3
"""Timeline of the split-K cluster decode GEMVs inside the real decode graph
(eet_debug_cltrace, CTA 0 and the last CTA of each launch): per launch, us
relative to the previous traced launch's end: [start, wait passed, X staged,
weights landed, partials sent, end]; then medians per (N, K)."""
import ctypes as C, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402
from paper_2104_12470_b200 import _lib  # noqa: E402


def main():
    b = int(os.environ.get("B", "16"))
    dt = os.environ.get("DT", "fp16")
    cfg = eet.ModelConfig(b, 1024, 24, 16, 512, 1024, datatype_label=dt)
    w = eet.random_weights(cfg, 50257, seed=0)
    rng = np.random.default_rng(0)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=512)] for _ in range(b)]
    req = eet.GenerationRequest(prompts=prompts, steps=6)
    pool = eet.BufferPool()
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    _lib.lib().eet_debug_cltrace(1, None, None)
    eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
    out = np.zeros((8192, 24), dtype=np.int64); n = C.c_int()
    _lib.lib().eet_debug_cltrace(0, out.ctypes.data_as(C.c_void_p), C.byref(n))
    r = out[:n.value]
    cycles(r)
    # one record per launch: the CTA with the later end
    key = r[:, 0]
    order = np.argsort(r[:, 2], kind="stable")
    r = r[order]
    launches = []
    i = 0
    while i < len(r):
        j = i + 1
        while j < len(r) and r[j, 0] == r[i, 0] and abs(r[j, 2] - r[i, 2]) < 3000 and j - i < 2:
            j += 1
        grp = r[i:j]
        launches.append((grp[0, 0], grp[:, 2].min(), grp[:, 3].max(), grp[:, 4].max(), grp[:, 5].max(),
                         grp[:, 6].max(), grp[:, 7].max()))
        i = j
    L = np.array(launches, dtype=np.int64)
    names = {}
    rows = []
    for k in range(1, len(L)):
        prev_end = L[k - 1, 6]
        rel = (L[k, 1:] - prev_end) / 1e3
        nk = L[k, 0]
        tag = f"N{nk >> 32} K{(nk & 0xffffffff) >> 1}{' LN' if nk & 1 else ''}"
        rows.append((tag, rel))
    print("one layer of a middle decode step (us rel. to previous traced launch end):")
    mid = len(rows) // 2
    for tag, rel in rows[mid:mid + 12]:
        print(f"  {tag:18s} " + " ".join(f"{v:7.2f}" for v in rel))
    print("medians per kind: start wait staged wready sent end (rel. prev end); own: end-wait")
    for tag in sorted(set(t for t, _ in rows)):
        sel = np.array([rel for t, rel in rows if t == tag])
        med = np.median(sel, axis=0)
        print(f"  {tag:18s} x{len(sel):4d} " + " ".join(f"{v:7.2f}" for v in med) +
              f"   own {np.median(sel[:, 5] - sel[:, 1]):.2f}")


def cycles(r):
    names = ["wait", "xload", "shfl", "clwait", "clsync", "staged", "wready", "mma", "sent", "clsync2", "end"]
    print("CTA-0 cycles since kernel start (median) per phase end:", " ".join(names))
    for key in sorted(set(r[:, 0])):
        sel = r[(r[:, 0] == key) & (r[:, 1] == 0)]
        med = np.median(sel[:, 8:19], axis=0)
        tag = f"N{key >> 32} K{(key & 0xffffffff) >> 1}{' LN' if key & 1 else ''}"
        gt = np.median(sel[:, 7] - sel[:, 2]) / 1e3
        print(f"  {tag:18s} x{len(sel):4d} " + " ".join(f"{v:7.0f}" for v in med) + f"   (gt {gt:.2f} us, "
              f"{(med[-1]) / max(gt, 1e-9) / 1e3:.2f} GHz)")


if __name__ == "__main__":
    main()
