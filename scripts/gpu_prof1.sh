cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -15
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 1 -c 2 -o gpurun_out/prof_spmv python scripts/prof_solve.py kernels > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_setup_solve.csv python scripts/prof_solve.py solve > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
