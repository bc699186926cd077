#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_round_check.sh r02p
timeout 900 python tools/r02/e2e_phases.py > gpurun_out/r02p_e2e_phases.txt 2>&1
