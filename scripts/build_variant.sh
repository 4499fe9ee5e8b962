#!/bin/bash
# Build a library variant with extra nvcc defines: bash scripts/build_variant.sh NAME "-DFOO=1 ..."
# -> abvariants/libmoe_NAME.so (for scripts/gpu_variant_ab.sh)
set -e
NAME=$1; EXTRA=$2
D=/tmp/bv_$NAME; mkdir -p $D abvariants
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $EXTRA"
rm -f $D/*.o
pids=()
for f in paper_2211_15841_b200/csrc/*.cu; do
  b=$(basename $f .cu); $NV -c $f -o $D/$b.o &
  pids+=($!)
done
for pid in "${pids[@]}"; do wait $pid || { echo "compile failed"; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o abvariants/libmoe_$NAME.so $D/*.o
echo built abvariants/libmoe_$NAME.so
