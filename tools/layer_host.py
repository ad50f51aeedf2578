#!/usr/bin/env python3
"""Host vs device time of one prompt-phase layer call (decoder_layer_forward
on CUDA tensors) at a layer workload: wall clock per call over 200 calls
(one sync at the end) and CUDA-event device time over the same calls."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2104_12470_b200 as eet  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = dict(bench.WORKLOADS[wl])
lens = bench.lengths_for(w)
desc = eet.make_batch(lens)
s = desc.seq_len
cfg = eet.ModelConfig(batch_size=w["batch"], hidden_size=w["hidden"], layer_count=1, head_count=w["heads"],
                      max_prompt=s, max_sequence=s, datatype_label=w["dtype"])
lw = eet.random_weights(eet.ModelConfig(1, w["hidden"], 1, w["heads"], 1, 1), 8, seed=0).layers[0]
kv, acts = eet.preallocate_caches(cfg)
pool = eet.BufferPool()
x = torch.randn(w["batch"], s, w["hidden"], device="cuda")


def step():
    kv._filled = 0
    eet.decoder_layer_forward(x, lw, kv, desc, eet.Phase.PROMPT_PARALLEL, pool, acts, 0)


for _ in range(5):
    step()
torch.cuda.synchronize()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(n):
    step()
e1.record()
t_host = (time.perf_counter() - t0) / n * 1e6
torch.cuda.synchronize()
print(f"{wl}: host issue {t_host:.1f} us/call, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/call")
