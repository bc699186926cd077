#!/bin/bash
# tcgen05 Gram: tests + probe; sharded world-1 vs single (r02bb); cfg5 loop probe
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q -k "gram_tf32x3" > gpurun_out/r02cc_pytest_gram.log 2>&1; echo rc=$? >> gpurun_out/r02cc_pytest_gram.log
timeout 300 python tools/r02/gram_tc_probe.py > gpurun_out/r02cc_gram_probe.txt 2>&1; echo rc=$? >> gpurun_out/r02cc_gram_probe.txt
timeout 900 python -m pytest tests/test_gpu_rsvd_svt.py -x -q -k "fp32" > gpurun_out/r02cc_pytest_fp32.log 2>&1; echo rc=$? >> gpurun_out/r02cc_pytest_fp32.log
bash tools/r02/r02bb.sh > gpurun_out/r02cc_bb.txt 2>&1
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 2000 python tools/r02/cfg5_svt_probe.py > gpurun_out/r02cc_cfg5_svt.txt 2>&1; echo rc=$? >> gpurun_out/r02cc_cfg5_svt.txt
