#!/bin/bash
# compute-sanitizer restricted to the fused decode kernels (qkv_attn_o,
# attn_o) and the decode GEMVs / LM head, on the fused-decode tests; logs in
# gpurun_out/
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
F="--kernel-name kns=qkv_attn_o --kernel-name kns=attn_o --kernel-name kns=gemv_cl --kernel-name kns=lm_head"
timeout 900 compute-sanitizer --tool racecheck $F --print-limit 20 python -m pytest tests/test_attn_o_gpu.py -x -q -p no:cacheprovider > gpurun_out/racecheck_fused.log 2>&1
echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/racecheck_fused.log | head -4
timeout 900 compute-sanitizer --tool synccheck $F --print-limit 20 python -m pytest tests/test_attn_o_gpu.py -x -q -p no:cacheprovider > gpurun_out/synccheck_fused.log 2>&1
echo "synccheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/synccheck_fused.log | head -4
timeout 900 compute-sanitizer --tool memcheck $F --leak-check no --print-limit 20 python -m pytest tests/test_attn_o_gpu.py tests/test_determinism_gpu.py -x -q -p no:cacheprovider > gpurun_out/memcheck_fused.log 2>&1
echo "memcheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck_fused.log | head -4
