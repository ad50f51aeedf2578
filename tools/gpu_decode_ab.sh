#!/bin/bash
# round-2 decode: correctness of the split-K cluster GEMV path, per-step time A/B, trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_headline_gpu.py tests/test_layer_gpu.py tests/test_acceptance_gpu.py -x -q -k "generate or criterion_3 or nan" -p no:cacheprovider > gpurun_out/r2_decode_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_decode_tests.log
(B=16 timeout 300 python tools/decode_step_time.py; EET_CL_WARM=0 B=16 timeout 300 python tools/decode_step_time.py; EET_GEMV_CL=0 B=16 timeout 300 python tools/decode_step_time.py;
 B=1 timeout 300 python tools/decode_step_time.py; EET_GEMV_CL=0 B=1 timeout 300 python tools/decode_step_time.py;
 timeout 300 python tools/cltrace.py) > gpurun_out/r2_decode_time.log 2>&1
