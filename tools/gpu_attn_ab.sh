# A/B of the prefill attention launch order (work list vs grid order).
export PYTHONUNBUFFERED=1
timeout 150 python -m pytest tests/test_layer_gpu.py -m gpu -x -q -p no:cacheprovider -k "16bit" 2>&1 | tail -3 || exit 1
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for w in c3 c4; do
  for v in list grid; do
    if [ $v = grid ]; then export EET_ATTN_GRID=1; else unset EET_ATTN_GRID; fi
    timeout 200 python bench.py --workload $w --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$w $v', d['ms_per_step'], d['value'])"
  done
done
unset EET_ATTN_GRID
timeout 300 python tools/layer_profile.py --workload c3 2>&1 | tail -12
