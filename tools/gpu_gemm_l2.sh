# A/B of the tcgen05 GEMM L2 plan (EET_GEMM_L2: 0 previous, 1 A evict-last +
# K-sized groups, 2 normal policies + K-sized groups), plus the fp32 GEMM.
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for w in c3 c4 c5; do
  for v in 0 1 2 0 1 2; do
    EET_GEMM_L2=$v timeout 200 python tools/layer_profile.py --workload $w --reps 3 --time 2>&1 | grep gemm_tc | sed "s/^/$v /"
  done
done
timeout 200 python tools/layer_profile.py --workload c1 --reps 5 --time 2>&1
mkdir -p gpurun_out/l2
for v in 0 1; do
  EET_GEMM_L2=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:gemm_tc --log-file gpurun_out/l2/c4_$v.csv python tools/layer_profile.py --workload c4 > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/l2/c4_$v.csv | sed "s/^/ncu c4 mode $v: /"
done
