#!/bin/bash
mkdir -p gpurun_out
LR_GEMM_TILE=6 timeout 600 python tools/r02/gemm_tma_probe.py > gpurun_out/r02z_gemm.txt 2>&1
LR_NATIVE_LIB=build_var/gemm2/liblowrank_b200.so LR_GEMM_TILE=6 timeout 600 python tools/r02/gemm_tma_probe.py 2>&1 | sed 's/tile=6/tile=6-minb2/' >> gpurun_out/r02z_gemm.txt
