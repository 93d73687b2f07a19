# A/B of the coarse tail: per-level graph kernels vs the grid-cooperative tail
# (cfg2 bench solve times); MAMG_TAIL_CACHE=1 keeps coarsest rows in registers
cd $GRAFT_REPO_ROOT
run() { timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$1', 'solve', round(d['solve_s']*1e3,3), 'vcycle_us', round(d['vcycle']['ms']*1e3,1))"; }
for r in 1 2; do
  MAMG_TAIL_ROWS=0 run "per-level                 "
  MAMG_TAIL_ROWS=5000 MAMG_TAIL_GRID=1 MAMG_TAIL_CACHE=1 run "grid coarsest cached     "
  MAMG_TAIL_ROWS=20000 MAMG_TAIL_GRID=1 MAMG_TAIL_CACHE=1 run "grid tail <=20k cached   "
done
MAMG_TAIL_ROWS=5000 MAMG_TAIL_GRID=1 MAMG_TAIL_CACHE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pcg or cycle" 2>&1 | tail -2
