#!/bin/bash
# Build variant libraries of the line-aligned group kernels (launch-bounds min blocks, gathers in flight)
# into build_var/<name>/liblowrank_b200.so; run a probe against one with LR_NATIVE_LIB=...
set -e
build_one() {  # name, extra nvcc defines
  local name=$1; shift
  mkdir -p build_var/$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
    -c paper_1810_06860_b200/csrc/lr_sparse.cu -o build_var/$name/lr_sparse.o
  objs=$(ls build/*.o | grep -v lr_sparse.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_var/$name/liblowrank_b200.so $objs build_var/$name/lr_sparse.o -lm
}
# round 2, first sweep (profiles/r02k_group_kernel_variants.txt):
#   build_one minb3 -DLR_GRP_MINB=3; build_one q16 ...; build_one minb3q ...
# second sweep: the SVT kernel's occupancy against gathers in flight
for v in ${VARIANTS:-"svt2q4:-DLR_SVT_MINB=2 -DLR_SVT_Q3=4 -DLR_SVT_Q2=8" "svt2q2:-DLR_SVT_MINB=2" "svt4q1:-DLR_SVT_MINB=4 -DLR_SVT_Q3=1 -DLR_SVT_Q2=2 -DLR_SVT_Q1=4"}; do
  build_one ${v%%:*} ${v#*:}
done
