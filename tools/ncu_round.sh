#!/bin/bash
# ncu evidence for profiles/: launch lists (per-launch duration + DRAM bytes,
# cold-cache, serialised) of the c2 generate path and the c3/c4/c5 layers,
# plus one `--set full` capture of each dominant kernel. ONE GPU:
#   gpurun --timeout 2400 -- 'bash tools/ncu_round.sh'
# Outputs land in gpurun_out/ncu/ (scratch); summaries are copied to profiles/.
set -x
O=gpurun_out/ncu
mkdir -p $O
NCU=ncu
LIST="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
FULL="--set full --clock-control none --import-source on"

timeout 900 $NCU $LIST --log-file $O/launches_c2.csv python tools/decode_profile.py --steps 4 > $O/launches_c2.log 2>&1
for w in c3 c4 c5; do
  timeout 600 $NCU $LIST --log-file $O/launches_$w.csv python tools/layer_profile.py --workload $w > $O/launches_$w.log 2>&1
done

# full captures of the top kernels (skip the warm-up call's launches)
timeout 600 $NCU $FULL -k regex:gemv_cl -s 400 -c 4 -o $O/gemv_cl_c2 -f python tools/decode_profile.py --steps 4 > $O/gemv_cl_c2.log 2>&1
timeout 600 $NCU $FULL -k regex:lm_head -s 3 -c 1 -o $O/lm_head_c2 -f python tools/decode_profile.py --steps 4 > $O/lm_head_c2.log 2>&1
timeout 600 $NCU $FULL -k regex:qkv_attn_o -s 60 -c 2 -o $O/qkv_attn_o_c2 -f python tools/decode_profile.py --steps 4 > $O/qkv_attn_o_c2.log 2>&1
timeout 600 $NCU $FULL -k regex:attn_tc -s 1 -c 1 -o $O/attn_tc_c3 -f python tools/layer_profile.py --workload c3 > $O/attn_tc_c3.log 2>&1
timeout 600 $NCU $FULL -k regex:gemm_tc -s 4 -c 4 -o $O/gemm_tc_c4 -f python tools/layer_profile.py --workload c4 > $O/gemm_tc_c4.log 2>&1
timeout 600 $NCU $FULL -k regex:attn_tc -s 1 -c 1 -o $O/attn_tc_c4 -f python tools/layer_profile.py --workload c4 > $O/attn_tc_c4.log 2>&1
ls -la $O
# summaries on the box; the .ncu-rep files are too large to bring back
for r in $O/*.ncu-rep; do python tools/ncu_summary.py full $r > ${r%.ncu-rep}.full.txt 2>&1; done
for w in c2 c3 c4 c5; do python tools/ncu_summary.py launches $O/launches_$w.csv > $O/launches_$w.txt 2>&1; done
python tools/traffic_update.py $O > $O/traffic_update.log 2>&1
rm -f $O/*.ncu-rep
gzip -f $O/launches_c2.csv
