#!/bin/bash
# prompt-GEMM epilogue A/B: c3/c4/c5 layer lines + ncu of the c4 GEMMs (tensor-pipe activity per launch)
mkdir -p gpurun_out
: > gpurun_out/gemm_ab.log
for w in c3 c4 c5; do
  timeout 400 python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/gemm_ab_$w.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/gemm_ab_$w.json')); print('$w', round(d['ms_per_step'],3), d['kernels'].get('gemm_tc'))" >> gpurun_out/gemm_ab.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:gemm_tc --csv python tools/layer_profile.py --workload c4 > gpurun_out/gemm_ab_ncu.csv 2>&1
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_baseline_layers_gpu.py -q -p no:cacheprovider -x -k "tensor_core_gemm or c3 or c4" >> gpurun_out/gemm_ab.log 2>&1
