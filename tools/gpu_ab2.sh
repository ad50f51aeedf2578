timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 --timeout-method thread 2>&1 | tail -1
for i in 1 2; do
for v in 0 1; do EET_ATTN_POLY=$v timeout 300 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('poly=$v c4', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items() if k=='attn_prefill'})"; done
for v in 0 1; do EET_ATTN_POLY=$v timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('poly=$v c3', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items() if k=='attn_prefill'})"; done
done
