#!/bin/bash
# Round-end check after the GEPP moved to one CTA per SM: reproducers, GPU tests, both bench arms, smoke
mkdir -p gpurun_out
timeout 400 python tools/r02/omega_determinism.py 3000 32 2>&1 | tail -1 | cut -c1-300
timeout 400 python tools/r02/omega_determinism.py 2000 48 2>&1 | tail -1 | cut -c1-300
timeout 400 python tools/r02/bki_determinism.py 1500 2>&1 | grep "omega=" | cut -c1-300
(time timeout 1800 python -m pytest tests -m gpu -x -q) > gpurun_out/r02bn_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02bn_pytest_gpu.log | head -2
(time timeout 900 python bench.py --impl reference) > gpurun_out/r02bn_ref.log 2>&1; echo "ref rc=$?"
(time timeout 1200 python bench.py) > gpurun_out/r02bn_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python __graft_entry__.py > gpurun_out/r02bn_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02bn_smoke.log
timeout 900 python bench.py --shard --cpu-baseline skip --extras off > gpurun_out/r02bn_shard.log 2>&1; echo "shard rc=$?"
