# tcgen05 GEMM raster-group sweep (EET_GEMM_PANEL_MB: A-panel budget in MB)
export PYTHONUNBUFFERED=1
for w in c3 c4 c5; do
  for v in 20 40 64 96 20 40 64 96; do
    EET_GEMM_PANEL_MB=$v timeout 200 python tools/layer_profile.py --workload $w --reps 3 --time 2>&1 | grep gemm_tc | sed "s/^/$v /"
  done
done
