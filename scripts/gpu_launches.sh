# ncu launch lists (time + DRAM bytes) of one setup + solve per spec, aggregated per kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in ${SPECS:-randk3d:160,160,160,0 aniso27:128,128,128,0.01 elast3d:100,100,100}; do
  tag=$(echo $spec | cut -d: -f1)
  SPEC=$spec timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python scripts/prof_solve.py solve \
    > gpurun_out/launches_$tag.log 2>&1
  echo "== $spec rc=$?"
  python scripts/launch_breakdown.py gpurun_out/launches_$tag.csv 25 | tee gpurun_out/launches_$tag.txt
done
