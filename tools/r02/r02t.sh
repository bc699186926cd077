#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_round_check.sh r02t
timeout 600 python tools/r02/cfg4_timeline.py > gpurun_out/r02t_timeline.txt 2>&1
python -c "import sys; sys.path.insert(0,'.')
from paper_1810_06860_b200 import rsvd; print(rsvd.REUSE_STATS)" >> gpurun_out/r02t_timeline.txt 2>&1
