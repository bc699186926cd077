#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/r02/gemm_tma_probe.py > gpurun_out/r02x_gemm.txt 2>&1
LR_GEMM_TILE=6 timeout 600 python tools/r02/gemm_tma_probe.py >> gpurun_out/r02x_gemm.txt 2>&1
LR_NATIVE_LIB=build_var/gemm2/liblowrank_b200.so LR_GEMM_TILE=6 timeout 600 python tools/r02/gemm_tma_probe.py 2>&1 | sed 's/tile=6/tile=6-minb2/' >> gpurun_out/r02x_gemm.txt
LR_GEMM_TILE=6 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02x_pytest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_pytest_tma.log
