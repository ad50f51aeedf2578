# quick GPU check: parity tests + layer benches
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 --timeout-method thread > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log | cut -c1-300
for w in ${WL:-c3 c4 c5}; do timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', round(d['value']), 'ms/step', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"; done
