#!/bin/bash
mkdir -p gpurun_out
(echo "== cl, no PDL"; EET_NO_PDL=1 timeout 300 python tools/cltrace.py | tail -6;
 echo "== packed, no PDL (ktrace)"; EET_NO_PDL=1 EET_GEMV_CL=0 timeout 300 python tools/ktrace.py;
 echo "== step times no PDL: cl, packed"; EET_NO_PDL=1 B=16 timeout 300 python tools/decode_step_time.py; EET_NO_PDL=1 EET_GEMV_CL=0 B=16 timeout 300 python tools/decode_step_time.py) > gpurun_out/r2_trace2.log 2>&1
