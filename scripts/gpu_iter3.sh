# parity (all GPU tests) + cfg2 bench + cfg3/cfg5 benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
for c in ${CFGS:-cfg2 cfg3 cfg5}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c rc=$?"; tail -3 gpurun_out/bench_$c.err; python - <<PY
import json; d=json.load(open("gpurun_out/bench_$c.json"))
print({k:d[k] for k in ("value","setup_s","solve_s","iterations")}, "e2e", d["e2e"], "roof", round(d["roofline"]["frac"],3), d["roofline"]["ms_per_launch"], "spmv", d["spmv"], "vcyc", d["vcycle"])
PY
done
