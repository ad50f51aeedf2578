#!/bin/bash
# prefill attention A/B: parity tests, then c3/c4 layer lines with P through TMEM (default) vs smem
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_baseline_layers_gpu.py tests/test_acceptance_gpu.py -q -p no:cacheprovider -x -k "16bit or c3 or c4 or overflow or nan or generate" > gpurun_out/attn_ab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/attn_ab_tests.log
for w in c3 c4 c5; do
  for v in 1 0; do
    EET_ATTN_PTMEM=$v timeout 400 python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/attn_ab_${w}_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/attn_ab_${w}_$v.json')); print('$w ptmem=$v', round(d['ms_per_step'],3), d['kernels'].get('attn_prefill'))" >> gpurun_out/attn_ab.log
  done
done
