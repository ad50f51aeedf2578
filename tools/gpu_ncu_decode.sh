#!/bin/bash
O=gpurun_out/ncu_r2
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_cl -s 200 -c 4 -o $O/gemv_cl -f python tools/decode_profile.py --steps 4 > $O/gemv_cl.log 2>&1
ncu -i $O/gemv_cl.ncu-rep --page details --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy --section SpeedOfLight --section MemoryWorkloadAnalysis > $O/gemv_cl_details.txt 2>&1
ncu -i $O/gemv_cl.ncu-rep --page raw --csv --metrics smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_membar,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_sample_count,gpu__time_duration.sum,dram__bytes_read.sum > $O/gemv_cl_raw.csv 2>&1
rm -f $O/*.ncu-rep
