#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/r02/mem_probe.py > gpurun_out/r02y_mem.txt 2>&1
bash tools/r02/r02x.sh
