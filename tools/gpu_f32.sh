export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fp32 or c1 or golden or generate_fp32" 2>&1 | tail -2
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 200 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('c1', round(d['ms_per_step'],3), {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
