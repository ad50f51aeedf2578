export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 --timeout-method thread 2>&1 | tail -2
timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
B=1 timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
EET_SKIP=qkv,attn,o,w1,w2 timeout 200 python tools/decode_step_time.py | sed "s/^/tail-only /"
