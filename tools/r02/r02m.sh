#!/bin/bash
mkdir -p gpurun_out
tag=${1:-r02m}
for f in 1e-300 1e-13 1e-7; do LR_DENSE_NULL_FLOOR=$f timeout 300 python tools/r02/tcrq_probe.py >> gpurun_out/${tag}_tcrq.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "oracle_svd or clusters or group_kernel" > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
