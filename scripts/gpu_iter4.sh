cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for r in 1 2; do
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_$r.json 2> gpurun_out/bench_cfg2_$r.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg2_$r.json')); print(d['value'], d['step_ms'], d['setup_ms_steps'], d['solve_ms_steps'], d['e2e'])"
done
uptime; nproc
