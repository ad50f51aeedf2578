# round measurement: tests, smoke, bench lines for all workloads, ncu evidence
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 120 --timeout-method thread > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5; do timeout 400 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
for w in c1 c2 c3 c4 c5; do python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), 'cpu', (d.get('cpu_baseline') or {}).get('value'), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"; done
cat gpurun_out/bench_ref_c2.json | cut -c1-300
bash tools/ncu_round.sh > /dev/null 2>&1
ls gpurun_out/ncu | head -30
