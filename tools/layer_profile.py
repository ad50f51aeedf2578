#!/usr/bin/env python3
"""One prompt-phase decoder layer at a BASELINE layer workload (c1/c3/c4/c5)
for ncu captures: a warm-up call, then `--reps` calls. Select launches with
ncu -k/-s/-c, e.g.

  ncu --set full --clock-control none -k regex:attn_tc -s 1 -c 1 \
      -o gpurun_out/attn_c3 python tools/layer_profile.py --workload c3
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2104_12470_b200 as eet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3", choices=["c1", "c3", "c4", "c5"])
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--time", action="store_true", help="print per-kernel-kind event times of the reps")
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    lens = bench.lengths_for(w)
    desc = eet.make_batch(lens)
    s = desc.seq_len
    cfg = eet.ModelConfig(w["batch"], w["hidden"], 1, w["heads"], s, s, datatype_label=w["dtype"])
    lw = eet.random_weights(eet.ModelConfig(1, w["hidden"], 1, w["heads"], 1, 1), 8, seed=0).layers[0]
    kv, acts = eet.preallocate_caches(cfg)
    pool = eet.BufferPool()
    x = torch.from_numpy(np.random.default_rng(1).normal(0, 1, size=(w["batch"], s, w["hidden"]))
                         .astype(np.float32)).cuda()
    from paper_2104_12470_b200 import _lib
    for r in range(1 + a.reps):
        if a.time and r == 1:
            torch.cuda.synchronize()
            _lib.profile_enable(True)
        kv._filled = 0
        eet.decoder_layer_forward(x, lw, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    torch.cuda.synchronize()
    if a.time:
        for k, (n, ms, by, fl) in sorted(_lib.profile_summary().items(), key=lambda kv_: -kv_[1][1]):
            print(f"{a.workload} {k:16s} n={n:4d} us/launch={1e3 * ms / max(n, 1):9.2f} "
                  f"TFLOP/s={fl / max(ms, 1e-9) / 1e9:7.1f} GB/s={by / max(ms, 1e-9) / 1e6:7.1f}")


if __name__ == "__main__":
    main()
