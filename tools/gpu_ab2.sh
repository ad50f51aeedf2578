timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "tensor_core" 2>&1 | tail -1
for w in c3 c5 c4; do timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$w', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"; done
