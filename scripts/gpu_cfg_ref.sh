# full-size cfg 3-5 bench lines WITH the reference CPU baseline (long CPU runs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CFGS:-cfg3 cfg4 cfg5}; do
  timeout 3000 python bench.py --config $c --steps 3 > gpurun_out/bench_${c}_ref.json 2> gpurun_out/bench_${c}_ref.err
  echo "== $c rc=$?"; tail -2 gpurun_out/bench_${c}_ref.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_ref.json')); print(d['value'], d['e2e']['value'], d.get('cpu_baseline'), d.get('parity'))"
done
