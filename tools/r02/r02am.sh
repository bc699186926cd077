python -m pytest tests/test_gpu_kernels.py -x -q -k "omega_assembled" 2>&1 | tail -2
for cfg in "1 1" "0 1" "1 0"; do
  set -- $cfg
  LR_SUPERSET_DEVICE=$1 LR_OMEGA_SPEC_ESC=$2 python bench.py --cpu-baseline skip --extras off --e2e-steps 1 > gpurun_out/r02am_$1$2.log 2>&1
  python - <<XEOF
import json
for l in open("gpurun_out/r02am_$1$2.log"):
    if l.startswith("{"):
        d=json.loads(l); print("device=$1 esc=$2", round(d["value"],2), [round(x,1) for x in d["ms_per_job"]], round(d["e2e"]["value"],2), d["job_result"]["vs_reference_run"]["trace_identical"])
XEOF
done
LR_SUPERSET_DEVICE=1 timeout 600 python tools/r02/cfg4_timeline.py job > gpurun_out/r02am_timeline_dev.txt 2>&1; head -14 gpurun_out/r02am_timeline_dev.txt | cut -c1-140
