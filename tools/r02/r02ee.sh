#!/bin/bash
# session 3 re-entry: full GPU check of HEAD (tests, bench, smoke), tcgen05 Gram probe, sharded world-1 timeline
mkdir -p gpurun_out
bash tools/gpu_round_check.sh r02ee
timeout 300 python tools/r02/gram_tc_probe.py > gpurun_out/r02ee_gram_probe.txt 2>&1; echo rc=$? >> gpurun_out/r02ee_gram_probe.txt
SHARD=1 timeout 900 python tools/r02/cfg4_timeline.py job > gpurun_out/r02ee_shard_timeline.txt 2>&1; echo rc=$? >> gpurun_out/r02ee_shard_timeline.txt
timeout 600 python tools/r02/cfg4_timeline.py job > gpurun_out/r02ee_timeline.txt 2>&1; echo rc=$? >> gpurun_out/r02ee_timeline.txt
