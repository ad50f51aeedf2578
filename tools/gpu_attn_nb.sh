#!/bin/bash
# prefill attention work-list cost phases (EET_ATTN_NB) A/B at c3/c4/c5
mkdir -p gpurun_out
: > gpurun_out/attn_nb.log
for w in c3 c4 c5; do
  for nb in 4 2 1; do
    EET_ATTN_NB=$nb timeout 400 python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/attn_nb_${w}_$nb.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/attn_nb_${w}_$nb.json')); print('$w nb=$nb', round(d['ms_per_step'],3), d['kernels'].get('attn_prefill'))" >> gpurun_out/attn_nb.log
  done
done
timeout 300 env EET_ATTN_NB=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:attn_tc --csv python tools/layer_profile.py --workload c4 > gpurun_out/attn_nb_ncu.csv 2>&1
