#!/bin/bash
# GPU tests + group-kernel build variants (tools/r02/group_variants.sh) on the cfg4 SpMM / SVT-step probes
mkdir -p gpurun_out
tag=${1:-r02k}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
for v in default minb3 q16 minb3q; do
  if [ $v = default ]; then lib=""; else lib="LR_NATIVE_LIB=build_var/$v/liblowrank_b200.so"; fi
  echo "== $v" >> gpurun_out/${tag}_variants.txt
  env $lib timeout 600 python tools/spmm_cfg4_probe.py 11,22,45,66 >> gpurun_out/${tag}_variants.txt 2>&1
  env $lib RANKS=10,24,48,84 timeout 600 python tools/r02/svt_step_probe.py >> gpurun_out/${tag}_variants.txt 2>&1
done
tail -3 gpurun_out/${tag}_pytest_gpu.log
