export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 200 python tools/race_probe.py 2>&1 | head -1
timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
B=1 timeout 200 python tools/decode_step_time.py | sed "s/^/full /"
