set -x
timeout 700 python tools/hang_probe.py > gpurun_out/hang_probe.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 60 -k "not 16bit" > gpurun_out/gpu_tests_no16.log 2>&1
tail -5 gpurun_out/gpu_tests_no16.log
cat gpurun_out/hang_probe.txt
