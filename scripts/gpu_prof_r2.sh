# round-2 profile set (cfg 2): setup launch list, then ncu --set full of the
# steady-state triple dot / pair-2 reductions and the top setup kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_setup.csv python scripts/prof_setup.py > /dev/null 2>&1
echo "setup list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_blockdot<3" --launch-skip 10 -c 1 -o gpurun_out/ncu_dot3 python scripts/prof_solve.py solve > gpurun_out/ncu_dot3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpPcgPair2" --launch-skip 10 -c 1 -o gpurun_out/ncu_pair2 python scripts/prof_solve.py solve > gpurun_out/ncu_pair2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_suitor128|k_weights_cand|k_rowprod_warp" -c 3 -o gpurun_out/ncu_setup3 python scripts/prof_setup.py > gpurun_out/ncu_setup3.log 2>&1
echo done
