# A/B of setup time: default lib vs variant lib ($VAR) on a few specs
cd $GRAFT_REPO_ROOT
for spec in ${SPECS:-aniso27:128,128,128,0.01 elast3d:100,100,100 randk3d:160,160,160,0}; do
 for L in "" paper_1810_04221_b200/csrc/lib_${VAR}/libmamg_cuda.so; do
  SPEC=$spec TAG=${L:+$VAR} MAMG_LIB=$L REPS=${REPS:-8} timeout 600 python scripts/time_setup.py 2>&1 | tail -1
 done
done
