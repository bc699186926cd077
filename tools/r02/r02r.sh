#!/bin/bash
mkdir -p gpurun_out
for c in auto 32 48 64 96 128; do
  if [ $c = auto ]; then timeout 300 python tools/r02/wide_probe.py >> gpurun_out/r02r_wide.txt 2>&1;
  else LR_SPMM_CHUNK=$c timeout 300 python tools/r02/wide_probe.py >> gpurun_out/r02r_wide.txt 2>&1; fi
done
IMAX=3 timeout 400 python tools/r02/cfg4_defaults_probe.py > gpurun_out/r02r_cfg4_defaults.txt 2>&1
TMO=200 bash tools/r02/run_cfg4_dynamics.sh gpurun_out/r02r_cfg4_dynamics.txt
