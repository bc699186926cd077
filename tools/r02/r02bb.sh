#!/bin/bash
# sharded engine at world size 1 (collectives forced, NCCL) against the single-GPU engine, cfg4 job
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py -x -q > gpurun_out/r02bb_pytest_shards.log 2>&1; echo rc=$? >> gpurun_out/r02bb_pytest_shards.log
timeout 900 python bench.py --steps 2 --warmup 2 --extras off --cpu-baseline skip --e2e-steps 1 > gpurun_out/r02bb_single.json 2> gpurun_out/r02bb_single.err
timeout 900 python bench.py --shard --steps 2 --warmup 2 --extras off --cpu-baseline skip --e2e-steps 1 > gpurun_out/r02bb_shard.json 2> gpurun_out/r02bb_shard.err
python - <<'PY'
import json
for f in ("single", "shard"):
    try:
        d = json.loads(open(f"gpurun_out/r02bb_{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"], 2), "it/s", round(d["ms_per_step"], 1), "ms/job", d["iterations_per_job"],
              "e2e", round(d["e2e"]["value"], 2), d["job_result"]["residual"])
    except Exception as e:
        print(f, "failed", e)
PY
