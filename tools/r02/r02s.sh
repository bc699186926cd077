#!/bin/bash
# SVT kernel lane map: flat (bit-identical to the flat kernel) vs fit (fewest chunk slots)
mkdir -p gpurun_out
for mp in flat fit; do
  echo "== map $mp" >> gpurun_out/r02s_map.txt
  LR_SVT_MAP=$mp timeout 300 python tools/r02/tcrq_probe.py >> gpurun_out/r02s_map.txt 2>&1
  LR_SVT_MAP=$mp RANKS=10,17,24,33,48,64,84 timeout 600 python tools/r02/svt_step_probe.py >> gpurun_out/r02s_map.txt 2>&1
done
LR_SVT_MAP=fit timeout 1500 python -m pytest tests/test_gpu_rsvd_svt.py tests/test_gpu_shards.py -q > gpurun_out/r02s_pytest_fit.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_pytest_fit.log
LR_SVT_MAP=fit timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02s_timeline_fit.txt 2>&1
