cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
for d in _ab_head .; do
(cd $d && MAMG_BENCH_NO_CLOCKS=${NOCLK:-} timeout 900 python bench.py --config cfg2 --steps 8 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err; python -c "
import json; d=json.load(open('/tmp/b.json')); print('$d', round(d['value']*1e3,1), d['setup_ms_steps'], d['solve_ms_steps'], round(d['e2e']['value']*1e3,1))")
done; done
