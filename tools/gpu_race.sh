export PYTHONUNBUFFERED=1
timeout 600 compute-sanitizer --tool racecheck --print-limit 3 python tools/race_probe.py 2>&1 | grep -E "hazard|ERROR SUMMARY|per-op|megakernel" | head -8
echo ---
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "16bit and 768" 2>&1 | grep -E "hazard|ERROR SUMMARY|passed|failed" | head -8
echo ---
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_layer_gpu.py tests/test_decode_mk_gpu.py -x -q -p no:cacheprovider -k "16bit or generate or megakernel_matches or pad or cached or uneven" 2>&1 | grep -E "ERROR SUMMARY|passed|failed" | head -4
