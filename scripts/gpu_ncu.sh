# ncu --set full of matching kernels of one run (one GPU):
#   KREGEX='k_weights_cand' TAG=wc8 [SKIP=0] [COUNT=1] [SPEC=...] bash scripts/gpu_ncu.sh [setup|solve]
# report: gpurun_out/ncu_$TAG.ncu-rep (summaries: scripts/ncu_summary.py, scripts/ncu_lines.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
drv=scripts/prof_setup.py; arg=
[ "${1:-setup}" = solve ] && drv=scripts/prof_solve.py && arg=solve
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:$KREGEX" --launch-skip ${SKIP:-0} -c ${COUNT:-1} -o gpurun_out/ncu_$TAG -f \
  python $drv $arg > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
