export PYTHONUNBUFFERED=1
for i in 1 2; do
timeout 200 python tools/decode_step_time.py | sed "s/^/nbuf4 /"
EET_ATTN_NBUF6=1 timeout 200 python tools/decode_step_time.py | sed "s/^/nbuf6 /"
done
