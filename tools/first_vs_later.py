#!/usr/bin/env python3
"""The headline b1 fp16 generate run twice in one process, each run's
every-step logits against the teacher-forced fp32 oracle (norm-wise error),
plus where the two runs first differ."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2104_12470_b200 as eet  # noqa: E402
from oracle import eet_oracle as orc  # noqa: E402
from emu16 import norm_rel  # noqa: E402

steps = int(os.environ.get("STEPS", "64"))
cfg0 = eet.ModelConfig(16, 1024, 24, 16, 512, 1024)
W = eet.random_weights(cfg0, 50257, seed=0)
rng = np.random.default_rng(0)
prompts = [[int(t) for t in rng.integers(0, 50257, size=512)]]
cfg = eet.ModelConfig(1, 1024, 24, 16, 512, 1024, datatype_label="fp16")
runs = []
for r in range(int(os.environ.get("RUNS", "2"))):
    tr = eet.RunTrace(collect_logits=True)
    toks = eet.generate(W, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr)
    runs.append((toks, np.stack(tr.step_logits)))
for r, (toks, lg) in enumerate(runs):
    _, ref = orc.generate(W, prompts, steps, 512 + steps, collect_logits=True, forced=toks)
    ref = np.stack(ref)
    nr = [norm_rel(lg[s], ref[s]) for s in range(steps)]
    worst = int(np.argmax(nr))
    print(f"run {r}: worst norm-wise error {nr[worst]:.4f} at step {worst}; steps > 0.015: "
          f"{[s for s in range(steps) if nr[s] > 0.015][:10]}", flush=True)
    if r:
        d = np.abs(lg - runs[0][1]).max(axis=(1, 2))
        print(f"   vs run 0: " + ("identical" if not d.any() else f"first differs at step {int(np.argmax(d > 0))}"))
