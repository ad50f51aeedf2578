export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python -m pytest tests/test_layer_gpu.py tests/test_decode_mk_gpu.py -x -q -p no:cacheprovider -k "16bit or generate or megakernel_matches or pad or cached or uneven" > gpurun_out/memcheck.log 2>&1
echo "rc $?"; grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/memcheck.log | head -20
