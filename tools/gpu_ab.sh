export PYTHONUNBUFFERED=1
for sk in "" qkv attn o w1 w2; do EET_SKIP=$sk timeout 200 python tools/decode_step_time.py | sed "s/^/skip[$sk] /"; done
