# setup-time A/B: default build vs variant libs (MAMG_LIB), cfg2/cfg3 bench setup times
cd $GRAFT_REPO_ROOT
CS=paper_1810_04221_b200/csrc
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -1
for cfg in ${CFGS:-cfg2 cfg3}; do
  for r in 1 2; do
    for t in lib ${VARIANTS}; do
      MAMG_LIB=$CS/$t/libmamg_cuda.so timeout 300 python bench.py --config $cfg --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg $t', 'setup', round(d['setup_s']*1e3,3), 'solve', round(d['solve_s']*1e3,3))"
    done
  done
done
