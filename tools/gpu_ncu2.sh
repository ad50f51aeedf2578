mkdir -p gpurun_out/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/ncu/attn_tc_c4_v3 -f python tools/layer_profile.py --workload c4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f32 -s 4 -c 1 -o gpurun_out/ncu/gemm_f32_c1 -f python tools/layer_profile.py --workload c1 > /dev/null 2>&1
ls gpurun_out/ncu | grep -E "v3|f32"
