# ncu --set full of the first launch of selected setup kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cap() { # tag spec kernel-regex lib
  MAMG_LIB=$4 SPEC=$2 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$3" -c 1 -o gpurun_out/ncu_$1 -f python scripts/prof_setup.py > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?"
}
cap warp_r randk3d:160,160,160,0 "k_rowprod_warp" ""
cap wc8_r randk3d:160,160,160,0 "k_weights_cand<8>" ""
cap mid_a_old aniso27:128,128,128,0.01 "k_rowprod_mid" paper_1810_04221_b200/csrc/lib_old/libmamg_cuda.so
cap wc32_a aniso27:128,128,128,0.01 "k_weights_cand<32>" ""
