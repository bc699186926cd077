#!/bin/bash
# Launch list of the bench command plus one `ncu --set full` capture per hot kernel of
# tools/ncu_target.py (run on the GPU box).  Usage: tools/ncu_capture.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
python tools/ncu_target.py > gpurun_out/${tag}_target.log 2>&1 || exit 1
[ -z "$SKIP_LAUNCHES" ] && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --cpu-baseline skip --svt off --e2e-steps 0 > gpurun_out/${tag}_launches.log 2>&1
# name regex : launches to skip (first matching launch after the skip is captured)
KERNELS=${KERNELS:-"gemm_kernel:0|spmm_kernel:0|lu_kernel:0|tridiag_kernel:0|chol_coop_kernel:0|bisect_kernel:0"}
IFS='|' read -ra SPECS <<< "$KERNELS"
for spec in "${SPECS[@]}"; do
  k=${spec%:*}; skip=${spec##*:}
  short=$(echo "$k" | sed 's/[^A-Za-z0-9]/_/g' | cut -c1-40)_$skip${NCU_ONLY:+_$NCU_ONLY}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" \
      --launch-skip $skip -c 1 -o gpurun_out/${tag}_${short} python tools/ncu_target.py > gpurun_out/${tag}_${short}.log 2>&1
done
ls -la gpurun_out | tail -20
