# c2 decode path check: gpu tests for generate/decode + bench c2 + kernel launch list
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ncu
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 --timeout-method thread > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'b1', d.get('latency_b1_s'), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
tail -3 gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_c2.csv python tools/decode_profile.py --steps 4 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/ncu/launches_c2.csv | head -8
