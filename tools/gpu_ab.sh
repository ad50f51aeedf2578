export PYTHONUNBUFFERED=1
EET_SKIP=qkv,o,w1,w2 timeout 200 python tools/decode_step_time.py | sed "s/^/attn bulk /"
EET_ATTN_RANGE=1 EET_SKIP=qkv,o,w1,w2 timeout 200 python tools/decode_step_time.py | sed "s/^/attn range /"
EET_ATTN_RANGE=1 EET_ATTN_NOMERGE=1 EET_SKIP=qkv,o,w1,w2 timeout 200 python tools/decode_step_time.py | sed "s/^/attn range-nomerge /"
EET_SKIP=qkv,attn,o,w1,w2 timeout 200 python tools/decode_step_time.py | sed "s/^/none /"
