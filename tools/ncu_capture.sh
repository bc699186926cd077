#!/bin/bash
# One `ncu --set full` capture per hot kernel of tools/ncu_target.py (run on the GPU box).
# Usage: tools/ncu_capture.sh <tag>   -> gpurun_out/<tag>_<kernel>.ncu-rep
tag=${1:-r01}
mkdir -p gpurun_out
python tools/ncu_target.py > gpurun_out/${tag}_target.log 2>&1 || exit 1
for k in spmm_kernel lu_kernel gemm_kernel chol_coop_kernel tridiag_kernel sddmm_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/${tag}_$k python tools/ncu_target.py > gpurun_out/${tag}_$k.log 2>&1
done
ls -la gpurun_out
