# cfg 3-5: GPU parity tests + bench lines (no CPU baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -15
for c in ${CFGS:-cfg3 cfg4 cfg5}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c rc=$?"; tail -3 gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json
done
