# quick iteration: parity subset + bench + (optional) ncu of one kernel regex ($1)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
tail -3 gpurun_out/bench_iter.err; cat gpurun_out/bench_iter.json
if [ -n "$1" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -o gpurun_out/prof_iter python scripts/prof_solve.py kernels > gpurun_out/ncu_iter.log 2>&1
tail -2 gpurun_out/ncu_iter.log
fi
