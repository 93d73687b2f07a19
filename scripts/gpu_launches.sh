cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python scripts/prof_solve.py solve > gpurun_out/ncu_l.log 2>&1
tail -2 gpurun_out/ncu_l.log
