#!/bin/bash
# decode per-step time A/B (tools/decode_step_time.py): default vs env switches given as arguments
# usage: bash tools/gpu_decode_ab.sh "EET_X=1" "EET_Y=2 EET_Z=0" ...
mkdir -p gpurun_out
{
  B=16 timeout 300 python tools/decode_step_time.py
  for v in "$@"; do env $v B=16 timeout 300 python tools/decode_step_time.py; done
  B=1 timeout 300 python tools/decode_step_time.py
} > gpurun_out/decode_ab.log 2>&1
