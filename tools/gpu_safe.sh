export PYTHONUNBUFFERED=1
EET_DEBUG_LIB=1 timeout 120 python -m pytest tests/test_layer_gpu.py -x -q -p no:cacheprovider -k "16bit or generate" 2>&1 | grep -E "watchdog|passed|failed|Error" | head -5
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for w in c3 c4 c5; do timeout 120 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$w', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"; done
