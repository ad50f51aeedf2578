export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool racecheck --print-limit 100 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "16bit" > gpurun_out/racecheck_layers.log 2>&1
grep -E "passed|failed|RACECHECK SUMMARY" gpurun_out/racecheck_layers.log | tail -3
grep -oE "at void eet::[a-zA-Z_:]+<[^>(]*" gpurun_out/racecheck_layers.log | sort | uniq -c | sort -rn | head -10
timeout 600 compute-sanitizer --tool racecheck --print-limit 100 python tools/race_probe.py > gpurun_out/racecheck_decode.log 2>&1
grep -E "RACECHECK SUMMARY" gpurun_out/racecheck_decode.log | tail -2
grep -oE "at void eet::[a-zA-Z_:]+<[^>(]*" gpurun_out/racecheck_decode.log | sort | uniq -c | sort -rn | head -10
