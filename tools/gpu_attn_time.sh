# Per-kernel event times of the prompt-phase layer: prefill-attention
# schedules (EET_ATTN_NB cost phases, 0 = pure longest-first; grid order).
export PYTHONUNBUFFERED=1
for w in c3 c4 c5; do
  for v in 2 3 4 2 3 4; do
    if [ $v = grid ]; then export EET_ATTN_GRID=1; else unset EET_ATTN_GRID; export EET_ATTN_NB=$v; fi
    timeout 200 python tools/layer_profile.py --workload $w --reps 5 --time 2>&1 | grep attn | sed "s/^/$v /"
  done
done
