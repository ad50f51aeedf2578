#!/usr/bin/env python3
"""Which decode path drifts from the fp32 oracle (run under compute-sanitizer
to perturb timing): per-op graph path vs megakernel, fp16, small model."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12470_b200 as eet
from paper_2104_12470_b200 import _lib
from oracle import eet_oracle as orc

def run(mk, graph=True):
    prev = _lib.set_decode_megakernel(mk)
    tr = eet.RunTrace(collect_logits=True)
    toks = eet.generate(w, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr, use_graph=graph)
    _lib.set_decode_megakernel(prev)
    return toks, np.stack(tr.step_logits)

dt, b, h, heads, layers, vocab, steps = "fp16", 3, 256, 4, 2, 300, 8
rng = np.random.default_rng(b * 7 + h)
prompts = [[int(t) for t in rng.integers(0, vocab, size=int(n))] for n in rng.integers(3, 21, size=b)]
cfg = eet.ModelConfig(b, h, layers, heads, max(len(p) for p in prompts), max(len(p) for p in prompts) + steps, datatype_label=dt)
w = eet.random_weights(cfg, vocab, seed=h + layers)
ref_t, ref_l = orc.generate(orc.seeded_weights(h, layers, heads, vocab, cfg.max_sequence, h + layers), prompts, steps,
                            cfg.max_sequence, collect_logits=True)
ref_l = np.stack(ref_l)
for name, (t, l) in (("per-op graph", run(False)), ("per-op eager", run(False, False)), ("megakernel", run(True))):
    same = [bool(np.array_equal(t[:, s], ref_t[:, s])) for s in range(steps)]
    upto = same.index(False) if False in same else steps
    errs = [float(np.abs(l[s] - ref_l[s]).max()) for s in range(min(upto + 1, steps))]
    print(f"{name}: tokens agree with oracle for {upto} steps; max |dlogit| per step {['%.3f' % e for e in errs]}", flush=True)
