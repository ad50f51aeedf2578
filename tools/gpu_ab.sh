export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
timeout 200 python tools/decode_step_time.py | sed "s/^/cl4 /"
EET_GEMV_CL4=0 timeout 200 python tools/decode_step_time.py | sed "s/^/cl1 /"
done
B=1 timeout 200 python tools/decode_step_time.py | sed "s/^/cl4 /"
timeout 100 python tools/ktrace.py
