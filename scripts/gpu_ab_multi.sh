# A/B of setup + solve time across in-tree variant libraries (scripts/build_variant.sh <tag> "<defines>"):
#   VARS="tag1 tag2" [SPECS=...] bash scripts/gpu_ab_multi.sh   ("" = the default build)
cd $GRAFT_REPO_ROOT
for spec in ${SPECS:-randk3d:160,160,160,0 aniso27:128,128,128,0.01 elast3d:100,100,100}; do
 for V in "" $VARS; do
  L=${V:+paper_1810_04221_b200/csrc/lib_$V/libmamg_cuda.so}
  SPEC=$spec TAG=${V:-default} MAMG_LIB=$L REPS=${REPS:-8} timeout 600 python scripts/time_setup.py 2>&1 | tail -1
 done
done
