#!/bin/bash
# Omega draw variants on the cfg4 timeline; ncu of the line-aligned SpMM (w = 22) and SVT step (r = 10, 48)
mkdir -p gpurun_out
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02h_timeline.txt 2>&1
LR_OMEGA_SPEC=1 timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02h_timeline_spec1.txt 2>&1
LR_OMEGA_SPEC=0,1 timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02h_timeline_spec01.txt 2>&1
timeout 600 python tools/spmm_cfg4_probe.py 22 > gpurun_out/r02h_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_group -s 4 -c 2 -o gpurun_out/r02h_spmm22 python tools/spmm_cfg4_probe.py 22 > gpurun_out/r02h_ncu1.log 2>&1
NCU=1 RANKS=10,48 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/r02h_plain2.log 2>&1 && \
NCU=1 RANKS=10,48 timeout 900 ncu --set full --clock-control none --import-source on -k regex:svt_group2 -s 1 -c 3 -o gpurun_out/r02h_svt python tools/r02/svt_step_probe.py > gpurun_out/r02h_ncu2.log 2>&1
echo done
