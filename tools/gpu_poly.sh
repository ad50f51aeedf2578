# prefill softmax exp2: MUFU only (EET_ATTN_POLY=0) vs 3/8 FMA polynomial (1)
export PYTHONUNBUFFERED=1
for w in c4 c3 c5; do
  for v in 1 0 1 0; do
    EET_ATTN_POLY=$v timeout 200 python tools/layer_profile.py --workload $w --reps 5 --time 2>&1 | grep attn | sed "s/^/poly=$v /"
  done
done
