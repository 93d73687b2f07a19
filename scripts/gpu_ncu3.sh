# ncu --set full of selected kernels (first launch of each), summaries to gpurun_out
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in ${KERNELS:-k_blockdot k_suitor128 k_rowprod_warp}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_$k python scripts/prof_solve.py solve > gpurun_out/ncu_$k.log 2>&1
  echo "== $k rc=$?"; tail -1 gpurun_out/ncu_$k.log
  python scripts/ncu_summary.py gpurun_out/ncu_$k.ncu-rep > gpurun_out/ncu_$k.txt 2>&1; cat gpurun_out/ncu_$k.txt
done
