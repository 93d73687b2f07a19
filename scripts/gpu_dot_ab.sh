# A/B of the triple-dot CTA shape: MAMG_LIB points at variant builds (lib_<tag>)
cd $GRAFT_REPO_ROOT
CS=paper_1810_04221_b200/csrc
for r in 1 2; do
for t in lib_d82 lib lib_d44 lib_d42 lib_d63; do
  MAMG_LIB=$CS/$t/libmamg_cuda.so timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$t', 'solve', round(d['solve_s']*1e3,3), 'vcycle', round(d['vcycle']['ms'],4), 'it', d['iterations'], d['parity']['solution_bitwise_equal'] if 'parity' in d else '')"
done; done
for t in lib_d82 lib lib_d44 lib_d42 lib_d63; do
  echo "== $t"; MAMG_LIB=$CS/$t/libmamg_cuda.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_blockdot --launch-skip 20 --launch-count 4 python scripts/prof_solve.py solve 2>&1 | grep -E "OpTriple|duration" | grep -B1 duration | grep duration | head -2
done
