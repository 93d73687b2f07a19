# round checkpoint: full GPU suite, smoke, default bench (with the reference
# CPU baseline and per-level parity), the reference arm, the partitioned
# N=1 line, and the ncu launch list of one setup + solve (cfg 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r_gpu.txt
nproc >> gpurun_out/r_gpu.txt; lscpu | grep "Model name" >> gpurun_out/r_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err
timeout 900 python bench.py --partitioned --steps 3 > gpurun_out/r_bench_part.json 2> gpurun_out/r_bench_part.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r_launches.csv python scripts/prof_solve.py solve > /dev/null 2>&1
echo done
