bash tools/gpu_dec_ab.sh > gpurun_out/dec_ab.log 2>&1
cat gpurun_out/dec_ab.log
bash tools/gpu_round.sh
du -sh gpurun_out
