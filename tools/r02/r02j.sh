#!/bin/bash
# L1::no_allocate streams + L1 carve-out: GPU tests, SpMM / SVT-step probes, cfg4 timeline
mkdir -p gpurun_out
tag=${1:-r02j}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 600 python tools/spmm_cfg4_probe.py 11,16,22,33,45,66,132 > gpurun_out/${tag}_spmm.txt 2>&1
RANKS=10,24,48,84 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/${tag}_svt_step.txt 2>&1
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
timeout 600 python tools/spmm_cfg4_probe.py 22 > gpurun_out/${tag}_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_group -s 4 -c 1 -o gpurun_out/${tag}_spmm22 python tools/spmm_cfg4_probe.py 22 > gpurun_out/${tag}_ncu1.log 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log
