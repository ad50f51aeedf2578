#!/bin/bash
# compute-sanitizer on the decode path at HEAD (fused decode attention half
# qkv_attn_o / attn_o, split-K cluster GEMVs, LM head, decode attention) and
# the 16-bit layer path; logs in gpurun_out/
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
K="generate or criterion_3 or nan"
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python -m pytest tests/test_attn_o_gpu.py tests/test_decode_gemv_gpu.py tests/test_layer_gpu.py tests/test_acceptance_gpu.py -x -q -p no:cacheprovider -k "$K or decode or fused" > gpurun_out/memcheck_decode.log 2>&1
echo "memcheck rc $?"; grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/memcheck_decode.log | head -8
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_attn_o_gpu.py tests/test_decode_gemv_gpu.py tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "generate_graph or decode or fused" > gpurun_out/racecheck_decode.log 2>&1
echo "racecheck rc $?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/racecheck_decode.log | head -4
grep -oE "at void eet::[a-zA-Z_:]+<[^>(]*" gpurun_out/racecheck_decode.log | sort | uniq -c | sort -rn | head -10
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_attn_o_gpu.py tests/test_decode_gemv_gpu.py -x -q -p no:cacheprovider -k "not 8192" > gpurun_out/synccheck_decode.log 2>&1
echo "synccheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/synccheck_decode.log | head -4
