#!/bin/bash
# group2 SVT kernel on the flat lane map (bit-identical), 3 CTAs/SM: GPU tests, probes, cfg4 timeline
mkdir -p gpurun_out
tag=${1:-r02l}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
RANKS=10,24,48,84 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/${tag}_svt_step.txt 2>&1
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log
