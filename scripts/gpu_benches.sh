# bench lines: cfg2 (default, with CPU baseline) + cfg3/4/5 (no CPU baseline) + reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2_full.json 2> gpurun_out/bench_cfg2_full.err; tail -2 gpurun_out/bench_cfg2_full.err
cat gpurun_out/bench_cfg2_full.json
for c in cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > gpurun_out/bench_${c}_full.json 2> gpurun_out/bench_${c}_full.err; tail -2 gpurun_out/bench_${c}_full.err
  cat gpurun_out/bench_${c}_full.json
done
timeout 900 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref_full.json 2>/dev/null; cat gpurun_out/bench_ref_full.json
