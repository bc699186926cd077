#!/bin/bash
# GPU tests + cfg4 SpMM / SVT-step probes + cfg4 timeline after the line-aligned group kernels
mkdir -p gpurun_out
tag=${1:-r02g}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 600 python tools/spmm_cfg4_probe.py 11,16,22,33,45,66,132 > gpurun_out/${tag}_spmm.txt 2>&1
LR_SPMM_KERNEL=items timeout 600 python tools/spmm_cfg4_probe.py 22,45 >> gpurun_out/${tag}_spmm.txt 2>&1
RANKS=10,24,48,84,160 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/${tag}_svt_step.txt 2>&1
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log
