# megakernel: tests, phase trace, c2 bench
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_decode_mk_gpu.py -x -q -p no:cacheprovider > gpurun_out/mk_rel.log 2>&1
echo "rel rc $?"; tail -4 gpurun_out/mk_rel.log | cut -c1-400
EET_MK_TRACE=1 timeout 300 python tools/decode_profile.py --steps 16 2>&1 | grep -A1 "mk trace" | tail -6
timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'b1', d.get('latency_b1_s'), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
tail -3 gpurun_out/bench_c2.err
