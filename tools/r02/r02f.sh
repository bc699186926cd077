#!/bin/bash
# cfg4 timeline + host profile, SpMM / SVT-step probes, ncu of the cfg4 SpMM (w = 22) and SVT step (r = 48)
mkdir -p gpurun_out
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02f_timeline.txt 2>&1
timeout 600 python tools/r02/cfg4_timeline.py cprofile > gpurun_out/r02f_cprofile.txt 2>&1
timeout 600 python tools/spmm_cfg4_probe.py 11,16,22,33,45,66,132 > gpurun_out/r02f_spmm.txt 2>&1
RANKS=10,24,48,84 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/r02f_svt_step.txt 2>&1
timeout 600 python tools/spmm_cfg4_probe.py 22 > gpurun_out/r02f_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 4 -c 2 -o gpurun_out/r02f_spmm22 python tools/spmm_cfg4_probe.py 22 > gpurun_out/r02f_ncu1.log 2>&1
NCU=1 RANKS=48 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/r02f_plain2.log 2>&1 && \
NCU=1 RANKS=48 timeout 900 ncu --set full --clock-control none --import-source on -k regex:svt_flat -s 1 -c 1 -o gpurun_out/r02f_svt48 python tools/r02/svt_step_probe.py > gpurun_out/r02f_ncu2.log 2>&1
echo done
