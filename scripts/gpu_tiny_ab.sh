# tiny-level SpMV kernel A/B: per-sweep cost of the coarsest level and cfg1/2 solves
cd $GRAFT_REPO_ROOT
MAMG_SPMV_TINY=20000 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -1
for t in 0 5000 20000 70000; do
  echo "MAMG_SPMV_TINY=$t"; MAMG_SPMV_TINY=$t timeout 300 python scripts/sweep_cost.py 2>&1 | sed -n 2,5p
done
run() { timeout 300 python bench.py --config $1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$1 tiny=$MAMG_SPMV_TINY', 'solve', round(d['solve_s']*1e3,3), 'vcycle_us', round(d['vcycle']['ms']*1e3,1))"; }
for r in 1 2; do for t in 0 5000 20000; do export MAMG_SPMV_TINY=$t; run cfg1; run cfg2; done; done
