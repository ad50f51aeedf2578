export PYTHONUNBUFFERED=1
python tools/gemv_graph_bench.py 2>&1 | grep K4096
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 --timeout-method thread 2>&1 | tail -1
timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
EET_SKIP=w2 timeout 200 python tools/decode_step_time.py | sed "s/^/skip-w2 /"
B=1 timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
