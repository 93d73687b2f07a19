# BASELINE cfg 1, 3, 4, 5 bench lines (reference CPU baseline + per-level parity)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CFGS:-cfg1 cfg3 cfg4 cfg5}; do
  timeout 1500 python bench.py --config $c --steps 3 > gpurun_out/r_bench_$c.json 2> gpurun_out/r_bench_$c.err
  echo "$c rc=$?"
done
