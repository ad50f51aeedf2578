#!/usr/bin/env python3
"""Run-to-run determinism of generate (GPT-2-medium shape): the same fp16
request repeated, interleaved with bf16 / other-batch runs; logits must be
bit-identical every time (catches races in the decode kernels)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402

steps = int(os.environ.get("STEPS", "32"))
reps = int(os.environ.get("REPS", "8"))
cfg0 = eet.ModelConfig(16, 1024, 24, 16, 512, 512 + steps, datatype_label="fp16")
W = eet.random_weights(cfg0, 50257, seed=0)


def run(b, dt):
    cfg = eet.ModelConfig(b, 1024, 24, 16, 512, 512 + steps, datatype_label=dt)
    rng = np.random.default_rng(b)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=int(n))] for n in rng.integers(400, 513, size=b)]
    tr = eet.RunTrace(collect_logits=True)
    toks = eet.generate(W, eet.GenerationRequest(prompts=prompts, steps=steps), cfg, trace=tr)
    return toks, np.stack(tr.step_logits)


order = os.environ.get("ORDER", "")
if order:                                   # e.g. "1h,16b,1h,1h": batch + h (fp16) / b (bf16)
    ref = None
    for i, item in enumerate(order.split(",")):
        b, dt = int(item[:-1]), {"h": "fp16", "b": "bf16"}[item[-1]]
        t, l = run(b, dt)
        if b == 1 and dt == "fp16":
            if ref is None:
                ref = (t, l)
                print(f"{i} {item}: reference", flush=True)
            else:
                d = np.abs(l - ref[1]).max(axis=(1, 2))
                print(f"{i} {item}: " + ("identical" if not d.any() else
                      f"DIFFERS from step {int(np.argmax(d > 0))}, max |d| {d.max():.3g}"), flush=True)
        else:
            print(f"{i} {item}", flush=True)
    sys.exit(0)

ref = {b: run(b, "fp16") for b in (1, 16)}
bad = 0
for r in range(reps):
    run(16, "bf16")
    for b in (1, 16):
        t, l = run(b, "fp16")
        same = np.array_equal(t, ref[b][0]) and np.array_equal(l.view(np.int32), ref[b][1].view(np.int32))
        if not same:
            bad += 1
            d = np.abs(l - ref[b][1]).max(axis=(1, 2))
            print(f"rep {r} b{b}: DIFFERS, first step {int(np.argmax(d > 0))}, max |d| {d.max():.3g}", flush=True)
print(f"{bad} differing runs of {2 * reps}")
