set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01e_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r01e_bench.json 2> gpurun_out/r01e_bench.err; echo "bench rc=$?"
timeout 600 python __graft_entry__.py > gpurun_out/r01e_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r01e_pytest_gpu.log
