# sanitizers on the persistent prefill attention (parity cases with > 148 work items)
export PYTHONUNBUFFERED=1
K="lengths3 or lengths4"
timeout 900 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "$K" > gpurun_out/memcheck_attn.log 2>&1
echo "memcheck rc $?"; grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/memcheck_attn.log | head -8
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "$K" > gpurun_out/synccheck_attn.log 2>&1
echo "synccheck rc $?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/synccheck_attn.log | head -8
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "lengths3 and bf16" > gpurun_out/racecheck_attn.log 2>&1
echo "racecheck rc $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|passed|failed" gpurun_out/racecheck_attn.log | sort | uniq -c | head -12
