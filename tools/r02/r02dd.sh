#!/bin/bash
# tcgen05 Gram tests + probe, fp32-mode tests; sharded world-1 timeline; cfg5 loop (device-generated, delta 1)
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q -k "gram_tf32x3" > gpurun_out/r02dd_pytest_gram.log 2>&1; echo rc=$? >> gpurun_out/r02dd_pytest_gram.log
timeout 300 python tools/r02/gram_tc_probe.py > gpurun_out/r02dd_gram_probe.txt 2>&1; echo rc=$? >> gpurun_out/r02dd_gram_probe.txt
timeout 900 python -m pytest tests/test_gpu_rsvd_svt.py -x -q -k "fp32" > gpurun_out/r02dd_pytest_fp32.log 2>&1; echo rc=$? >> gpurun_out/r02dd_pytest_fp32.log
SHARD=1 timeout 900 python tools/r02/cfg4_timeline.py job > gpurun_out/r02dd_shard_timeline.txt 2>&1; echo rc=$? >> gpurun_out/r02dd_shard_timeline.txt
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 2000 python tools/r02/cfg5_svt_probe.py > gpurun_out/r02dd_cfg5_svt.txt 2>&1; echo rc=$? >> gpurun_out/r02dd_cfg5_svt.txt
