#!/bin/bash
# tf32x3 Gram with rotating accumulators: tests + probe; full GPU suite; cfg5 SVT loop (device generator, delta 1)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gram_tf32x3" > gpurun_out/r02ff_pytest_gram.log 2>&1; echo rc=$? >> gpurun_out/r02ff_pytest_gram.log
timeout 300 python tools/r02/gram_tc_probe.py > gpurun_out/r02ff_gram_probe.txt 2>&1; echo rc=$? >> gpurun_out/r02ff_gram_probe.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02ff_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ff_pytest_gpu.log
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 1800 python tools/r02/cfg5_svt_probe.py > gpurun_out/r02ff_cfg5_svt.txt 2>&1; echo rc=$? >> gpurun_out/r02ff_cfg5_svt.txt
