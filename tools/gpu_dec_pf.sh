# Decode attention: L2 bulk prefetch of the K/V range (EET_DEC_L2PF) A/B
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_layer_gpu.py tests/test_decode_mk_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for v in 1 0 1 0; do
  EET_DEC_L2PF=$v STEPS2=504 timeout 300 python tools/decode_step_time.py | sed "s/^/pf=$v /"
done
EET_DEC_L2PF=1 B=1 STEPS2=504 timeout 300 python tools/decode_step_time.py | sed "s/^/pf=1 /"
EET_DEC_L2PF=0 B=1 STEPS2=504 timeout 300 python tools/decode_step_time.py | sed "s/^/pf=0 /"
