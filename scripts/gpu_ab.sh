# A/B: default lib vs variant lib ($VAR), cfg2 + cfg3 bench kernels
cd $GRAFT_REPO_ROOT
for r in 1 2; do for L in "" paper_1810_04221_b200/csrc/lib_${VAR:-ns2}/libmamg_cuda.so; do
 for c in cfg2 cfg3; do
  MAMG_LIB=$L MAMG_BENCH_NO_CLOCKS=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('${L:-default}'[-30:], '$c', 'solve', round(d['solve_s']*1e3,2), 'smoother', round(d['roofline']['ms_per_launch']*1e3,1), 'us', round(d['roofline']['frac'],3), 'spmv', round(d['spmv']['ms']*1e3,1), round(d['spmv']['gbs']), 'vcyc', round(d['vcycle']['ms']*1e3,1))"
 done; done; done
