#!/bin/bash
# fused SVT step variants on the cfg4 pattern (tools/r02/svt_step_probe.py)
out=${1:-gpurun_out/r02_svt_step_variants.txt}
: > $out
export RANKS=${RANKS:-10,24,48,84,160,300}
LR_SVT_KERNEL=legacy SCATTER=1 python tools/r02/svt_step_probe.py >> $out 2>&1
python tools/r02/svt_step_probe.py >> $out 2>&1
for gt in ${GTS:-1,2,4 2,2,4 4,2,4 8,2,4 16,2,4 32,2,4 1,1,4 2,1,4 4,1,4 8,1,4 4,2,2 8,2,2 4,2,8 8,2,8 2,4,2 4,4,2 8,4,2 16,4,2 32,4,2}; do
  LR_SVT_FLAT=$gt python tools/r02/svt_step_probe.py >> $out 2>&1
done
