cd $GRAFT_REPO_ROOT
for cfg in "0 0" "40000 0" "40000 1" "70000 0" "300000 0"; do
  set -- $cfg
  MAMG_TAIL_ROWS=$1 MAMG_TAIL_CACHE=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('tail_rows=$1 cache=$2', 'setup',round(d['setup_s']*1e3,2),'solve',round(d['solve_s']*1e3,2),'vcycle_ms',round(d['vcycle']['ms'],4), 'steps', d['step_ms'])"
done
