cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
tail -3 gpurun_out/bench_iter.err; cat gpurun_out/bench_iter.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python scripts/prof_solve.py solve > gpurun_out/ncu_l.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 3 -c 1 -o gpurun_out/prof_chain python scripts/prof_solve.py solve > gpurun_out/ncu_c.log 2>&1
tail -1 gpurun_out/ncu_c.log
