#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_round_check.sh r02q
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02q_timeline.txt 2>&1
LR_OMEGA_SPEC=0 timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02q_timeline_spec0.txt 2>&1
