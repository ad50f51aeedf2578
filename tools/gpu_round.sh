# round measurement: tests, smoke, bench lines for all workloads, reference arm, ncu evidence
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ncu
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c5; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
bash tools/ncu_round.sh > /dev/null 2>&1
ls gpurun_out/ncu | head -40
