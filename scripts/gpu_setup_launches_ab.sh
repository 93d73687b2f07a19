# setup launch lists (default lib vs $VAR) per spec, top kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in ${SPECS:-aniso27:128,128,128,0.01 elast3d:100,100,100}; do
 tag=$(echo $spec | cut -d: -f1)
 for L in "" paper_1810_04221_b200/csrc/lib_${VAR}/libmamg_cuda.so; do
  t=${tag}_${L:+$VAR}
  MAMG_LIB=$L SPEC=$spec timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sl_$t.csv python scripts/prof_setup.py > /dev/null 2>&1
  echo "== $spec ${L:+$VAR}"; python scripts/launch_breakdown.py gpurun_out/sl_$t.csv 12
 done
done
