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
    for _ in range(1 + a.reps):
        kv._filled = 0
        eet.decoder_layer_forward(x, lw, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
