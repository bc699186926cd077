#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_round_check.sh r02v
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02v_timeline.txt 2>&1
RANKS=10,17,24,33,48,64,84 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/r02v_svt_step.txt 2>&1
