#!/usr/bin/env python3
"""Per-decode-step time of generate (c2 shape): (T(steps=S2) - T(steps=S1)) /
(S2 - S1), CUDA-event timed, median of 3. Development tool for A/B runs of
the decode path (env switches EET_NO_PACKED, EET_ATTN_RANGE, EET_MEGAKERNEL)."""
import os, sys, statistics
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_12470_b200 as eet  # noqa: E402

def main():
    b = int(os.environ.get("B", "16")); layers = int(os.environ.get("LAYERS", "24"))
    cfg = eet.ModelConfig(b, 1024, layers, 16, 512, 1024, datatype_label="fp16")
    w = eet.random_weights(cfg, 50257, seed=0)
    rng = np.random.default_rng(0)
    prompts = [[int(t) for t in rng.integers(0, 50257, size=512)] for _ in range(b)]
    pool = eet.BufferPool()
    def run(steps):
        req = eet.GenerationRequest(prompts=prompts, steps=steps)
        eet.generate(w, req, cfg, pool=pool); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); eet.generate(w, req, cfg, pool=pool); e.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(e))
        return statistics.median(ts)
    s2 = int(os.environ.get("STEPS2", "136"))
    t1, t2 = run(8), run(s2)
    tag = " ".join(f"{k}={os.environ[k]}" for k in ("EET_NO_PACKED", "EET_MEGAKERNEL", "EET_DEC_SPLITS", "EET_DEC_NBUF") if k in os.environ)
    print(f"b{b} L{layers} [{tag}] prompt+8: {t1:.2f} ms  per decode step (8..{s2}): {(t2 - t1) / (s2 - 8) * 1e3:.1f} us", flush=True)

if __name__ == "__main__":
    main()
