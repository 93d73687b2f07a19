# ncu (DRAM bytes + duration) of the level-0 solve kernels of one PCG iteration (cfg 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# skip the setup + first iterations, then capture ~one iteration's kernels
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_spmv_rows|k_smooth_zero|k_prolong_correct|k_blockdot|k_pcg_pair1" -s 400 -c 60 --csv \
  --log-file gpurun_out/ncu_kernels.csv python scripts/prof_solve.py solve > gpurun_out/ncu_kernels.log 2>&1
echo rc=$?
