#!/usr/bin/env python3
"""Uninitialised-read check for generate: the same b1 / b16 fp16 GPT-2-medium
generate run on a clean allocator and after the torch caching allocator was
filled with NaN / large values; logits and tokens must be bit-identical."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402


def run(b, dt, steps=24):
    cfg = eet.ModelConfig(b, 1024, 24, 16, 512, 512 + steps, datatype_label=dt)
    w = W[dt]
    rng = np.random.default_rng(1)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=int(n))] for n in rng.integers(400, 513, size=b)]
    tr = eet.RunTrace(collect_logits=True)
    toks = eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr)
    return toks, np.stack(tr.step_logits)


def poison(val):
    x = torch.empty(int(40e9) // 4, dtype=torch.float32, device="cuda")
    x.fill_(val)
    del x
    torch.cuda.synchronize()


cfg0 = eet.ModelConfig(16, 1024, 24, 16, 512, 536, datatype_label="fp16")
W = {"fp16": eet.random_weights(cfg0, 50257, seed=0)}
for b in (1, 16):
    t0, l0 = run(b, "fp16")
    for val in (float("nan"), 3.0e4, -1.0e30):
        poison(val)
        t1, l1 = run(b, "fp16")
        same = np.array_equal(t0, t1) and np.array_equal(l0.view(np.int32), l1.view(np.int32))
        d = np.abs(l0 - l1)
        print(f"b{b} poison {val}: identical {same}  max|dlogit| {np.nanmax(d):.3g}  nan {np.isnan(l1).sum()}", flush=True)
