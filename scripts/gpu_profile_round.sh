# round profile: bench launch list (one step after warm-up) + ncu full of the level-0 smoother
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4347 -c 1449 --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
echo "launch list rc=$?"
python scripts/launch_breakdown.py gpurun_out/bench_launches.csv 30 > gpurun_out/bench_launches.txt; head -20 gpurun_out/bench_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:EpiSmooth -c 1 -o gpurun_out/smoother_full python scripts/prof_solve.py kernels > gpurun_out/smoother_full.log 2>&1
echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/smoother_full.ncu-rep > gpurun_out/smoother_full.txt; cat gpurun_out/smoother_full.txt
