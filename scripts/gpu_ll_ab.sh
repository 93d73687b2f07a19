cd $GRAFT_REPO_ROOT
for L in "" paper_1810_04221_b200/csrc/lib_${VAR:-c4}/libmamg_cuda.so; do
  tag=$( [ -z "$L" ] && echo default || echo var )
  MAMG_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$tag.csv python scripts/prof_solve.py solve > /dev/null 2>&1
done
