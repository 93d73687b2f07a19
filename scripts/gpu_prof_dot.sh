cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:OpTriple -s 2 -c 1 -o gpurun_out/prof_triple python scripts/prof_solve.py solve > gpurun_out/ncu_t.log 2>&1
tail -1 gpurun_out/ncu_t.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_suitor -s 0 -c 1 -o gpurun_out/prof_suitor python scripts/prof_solve.py kernels > gpurun_out/ncu_s.log 2>&1
tail -1 gpurun_out/ncu_s.log
