# solve-time A/B: default build vs variant libraries (MAMG_LIB), cfg1-3 bench solve times
cd $GRAFT_REPO_ROOT
CS=paper_1810_04221_b200/csrc
for cfg in ${CFGS:-cfg1 cfg2 cfg3}; do
  for r in 1 2; do
    for t in lib ${VARIANTS}; do
      MAMG_LIB=$CS/$t/libmamg_cuda.so timeout 300 python bench.py --config $cfg --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg $t', 'solve', round(d['solve_s']*1e3,3), 'vcycle_us', round(d['vcycle']['ms']*1e3,1), 'setup', round(d['setup_s']*1e3,3))"
    done
  done
done
