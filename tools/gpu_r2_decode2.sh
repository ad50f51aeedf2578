#!/bin/bash
mkdir -p gpurun_out
(B=16 timeout 300 python tools/decode_step_time.py; EET_PDL_EARLY=1 B=16 timeout 300 python tools/decode_step_time.py; EET_PDL_EARLY=1 EET_CL_WARM=1 B=16 timeout 300 python tools/decode_step_time.py;
 EET_CL_NTMAX=16 B=16 timeout 300 python tools/decode_step_time.py; EET_CL_NTMAX=4 B=16 timeout 300 python tools/decode_step_time.py;
 for s in qkv attn o w1 w2 head; do EET_SKIP=$s B=16 timeout 300 python tools/decode_step_time.py; done) > gpurun_out/r2_decode_time2.log 2>&1
