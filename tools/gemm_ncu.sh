python tools/gemm_probe.py > gpurun_out/gemm_probe.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 2 -c 1 -o gpurun_out/gemm_syrk python tools/gemm_probe.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 26 -c 1 -o gpurun_out/gemm_nnup python tools/gemm_probe.py > /dev/null 2>&1
ls gpurun_out
