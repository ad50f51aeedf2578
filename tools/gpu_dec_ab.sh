# Decode attention A/B: splits per (sequence, head) x ring depth, per-step time
export PYTHONUNBUFFERED=1 STEPS2=504
timeout 200 python -m pytest tests/test_layer_gpu.py -m gpu -x -q -p no:cacheprovider -k "generate or 16bit" 2>&1 | tail -1
for cfg in "1 4" "2 3" "2 4" "3 3" "2 2" "1 4" "2 3"; do
  set -- $cfg
  EET_DEC_SPLITS=$1 EET_DEC_NBUF=$2 timeout 300 python tools/decode_step_time.py
done
