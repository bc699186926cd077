#!/bin/bash
# ncu --set full of the two sparse kernels on cfg4 (SpMM w = 22 / 45, SVT step r = 10 / 48 / 84); raw pages exported on the box
tag=${1:-r02ak}
mkdir -p gpurun_out
# full captures
timeout 600 python tools/spmm_cfg4_probe.py 22,45 > gpurun_out/${tag}_spmm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_group -s 4 -c 1 -o gpurun_out/${tag}_spmm22 python tools/spmm_cfg4_probe.py 22 > gpurun_out/${tag}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_group -s 4 -c 1 -o gpurun_out/${tag}_spmm45 python tools/spmm_cfg4_probe.py 45 > gpurun_out/${tag}_ncu1b.log 2>&1
NCU=1 RANKS=10,48,84 timeout 600 python tools/r02/svt_step_probe.py > gpurun_out/${tag}_svt_plain.log 2>&1 && \
NCU=1 RANKS=10,48,84 timeout 900 ncu --set full --clock-control none --import-source on -k regex:svt_group2 -c 6 -o gpurun_out/${tag}_svt python tools/r02/svt_step_probe.py > gpurun_out/${tag}_ncu2.log 2>&1
# the reports are too large to travel (64 MiB limit): export the raw pages here, keep only those
for f in gpurun_out/${tag}_spmm22 gpurun_out/${tag}_spmm45 gpurun_out/${tag}_svt; do
  ncu -i $f.ncu-rep --page raw --csv > $f.raw.csv 2>/dev/null
  rm -f $f.ncu-rep
done
ls -la gpurun_out | grep ${tag}
