#!/bin/bash
# prompt-GEMM A/B: c3/c4/c5 layer lines with an env switch off (A) and on (B),
# alternating, + ncu tensor-pipe activity of the c4 GEMMs for both, + tests.
#   SW=EET_GEMM_RESID_PIPE bash tools/gpu_gemm_ab.sh
SW=${SW:-EET_GEMM_RESID_PIPE}
mkdir -p gpurun_out
: > gpurun_out/gemm_ab.log
for rep in 1 2; do
  for v in 0 1; do
    for w in c3 c4 c5; do
      env $SW=$v timeout 400 python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/gemm_ab_$w.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/gemm_ab_$w.json')); print('$SW=$v', '$w', round(d['ms_per_step'],3), d['kernels'].get('gemm_tc'))" >> gpurun_out/gemm_ab.log
    done
  done
done
for v in 0 1; do
  env $SW=$v timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc --csv python tools/layer_profile.py --workload c4 > gpurun_out/gemm_ab_ncu_$v.csv 2>&1
done
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_baseline_layers_gpu.py tests/test_layer_gpu.py -q -p no:cacheprovider -x >> gpurun_out/gemm_ab.log 2>&1
tail -3 gpurun_out/gemm_ab.log
