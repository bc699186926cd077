#!/bin/bash
# Final check of the round: GPU tests, default bench (both arms), smoke, sharded world-1 bench, the ncu launch
# list of the bench command, ncu --set full of the two sparse kernels on cfg4 (SpMM w = 22 / 45, SVT step r = 10 / 48 / 84)
tag=${1:-r02ak}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
(time timeout 900 python bench.py --impl reference) > gpurun_out/${tag}_ref.log 2>&1; echo "ref rc=$?"
(time timeout 1200 python bench.py) > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python __graft_entry__.py > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py --shard --cpu-baseline skip --extras off > gpurun_out/${tag}_shard.log 2>&1; echo "shard rc=$?"
timeout 900 python bench.py --mode bki --cpu-baseline skip > gpurun_out/${tag}_bki.log 2>&1; echo "bki rc=$?"
# launch list of the bench command (svt headline only; the job is ~5500 launches)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 1 --warmup 1 --cpu-baseline skip --extras off --e2e-steps 0 > gpurun_out/${tag}_launches.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches_summary.txt 2>&1; head -12 gpurun_out/${tag}_launches_summary.txt
gzip -f gpurun_out/${tag}_launches.csv
ls -la gpurun_out | grep ${tag}
