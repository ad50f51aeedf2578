#!/bin/bash
mkdir -p gpurun_out
(timeout 300 python tools/cltrace.py; for s in qkv attn o w1 w2 head; do EET_SKIP=$s B=16 timeout 300 python tools/decode_step_time.py; done) > gpurun_out/r2_trace.log 2>&1
