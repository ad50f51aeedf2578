mkdir -p gpurun_out/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 400 -c 4 -o gpurun_out/ncu/gemv2 -f python tools/decode_profile.py --steps 4 > gpurun_out/ncu/gemv2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 60 -c 1 -o gpurun_out/ncu/attn_dec2 -f python tools/decode_profile.py --steps 4 > gpurun_out/ncu/attn_dec2.log 2>&1
tail -2 gpurun_out/ncu/gemv2.log
