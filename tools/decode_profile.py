#!/usr/bin/env python3
"""Short c2 generate (GPT-2-medium shape, fp16) for ncu captures: one warm-up
call, then one call with `--steps` decode steps. Use under ncu with -k/-s/-c
to select launches, e.g.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/decode_profile.py --steps 4
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2104_12470_b200 as eet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    cfg = eet.ModelConfig(a.batch, 1024, a.layers, 16, 512, 1024, datatype_label="fp16")
    w = eet.random_weights(cfg, 50257, seed=0)
    rng = np.random.default_rng(0)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=512)] for _ in range(a.batch)]
    req = eet.GenerationRequest(prompts=prompts, steps=a.steps)
    pool = eet.BufferPool()
    eet.generate(w, req, cfg, pool=pool, use_graph=not a.no_graph)
    torch.cuda.synchronize()
    eet.generate(w, req, cfg, pool=pool, use_graph=not a.no_graph)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
