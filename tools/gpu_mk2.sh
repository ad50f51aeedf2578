export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 6 -c 1 -o gpurun_out/ncu/mk_c2 -f python tools/decode_profile.py --steps 4 > gpurun_out/ncu/mk_c2.log 2>&1
tail -3 gpurun_out/ncu/mk_c2.log
