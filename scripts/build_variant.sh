# build an A/B variant of libmamg_cuda.so with extra nvcc defines into csrc/lib_<tag>/
# usage: scripts/build_variant.sh <tag> "-DFOO=1 ..."
set -e
ROOT=$(cd $(dirname $0)/.. && pwd)
CS=$ROOT/paper_1810_04221_b200/csrc
OUT=$CS/lib_$1; OBJ=$CS/build_$1
mkdir -p $OUT $OBJ/device $OBJ/capi
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O3,-msse4.2 -I$ROOT/include --expt-relaxed-constexpr $2"
for f in $CS/device/*.cu $CS/capi/*.cu; do
  rel=${f#$CS/}; $NV -dc $f -o $OBJ/${rel%.cu}.o &
done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $OBJ/device/*.o $OBJ/capi/*.o -o $OUT/libmamg_cuda.so -cudart static -lnccl
echo built $OUT/libmamg_cuda.so
