#!/bin/bash
# ncu --set full of the fused SVT step (svt_group2_kernel) on the cfg4 pattern at r = 10, 48, 84;
# sharded engine world-1 timeline after the device start / single-copy change
mkdir -p gpurun_out
for r in 10 48 84; do
  RANKS=$r NCU=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:svt_group2" \
     --launch-skip 1 -c 1 -o gpurun_out/r02gg_svt_r$r python tools/r02/svt_step_probe.py > gpurun_out/r02gg_svt_r$r.log 2>&1
done
for r in 10 48 84; do ncu -i gpurun_out/r02gg_svt_r$r.ncu-rep --page raw --csv > gpurun_out/r02gg_svt_r$r.raw.csv 2>/dev/null; done
SHARD=1 timeout 900 python tools/r02/cfg4_timeline.py job > gpurun_out/r02gg_shard_timeline.txt 2>&1; echo rc=$? >> gpurun_out/r02gg_shard_timeline.txt
IMAX=260 PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 1800 python tools/r02/cfg5_svt_probe.py > gpurun_out/r02gg_cfg5_svt.txt 2>&1; echo rc=$? >> gpurun_out/r02gg_cfg5_svt.txt
