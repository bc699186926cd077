#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02u_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02u_pytest_gpu.log
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02u_timeline.txt 2>&1
for v in default svt2q4 svt2q2 svt4q1; do
  if [ $v = default ]; then lib=""; else lib="LR_NATIVE_LIB=build_var/$v/liblowrank_b200.so"; fi
  echo "== $v" >> gpurun_out/r02u_svt_variants.txt
  env $lib RANKS=10,17,24,33,48,64,84 timeout 600 python tools/r02/svt_step_probe.py >> gpurun_out/r02u_svt_variants.txt 2>&1
done
tail -3 gpurun_out/r02u_pytest_gpu.log
