#!/bin/bash
# pre-start of the next inner SVD behind the fused step: SVT parity tests, cfg4 timeline; e2e phases
mkdir -p gpurun_out
tag=${1:-r02o}
timeout 1500 python -m pytest tests/test_gpu_rsvd_svt.py tests/test_gpu_shards.py -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/${tag}_timeline.txt 2>&1
LR_SVT_PRESTART=0 timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/${tag}_timeline_noprestart.txt 2>&1
timeout 900 python tools/r02/e2e_phases.py > gpurun_out/${tag}_e2e_phases.txt 2>&1
tail -3 gpurun_out/${tag}_pytest_gpu.log
