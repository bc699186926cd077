# Superset draw threads (device assembly on) and the default path, all pool threads otherwise
for cfg in "1 4" "1 6" "1 8" "1 12" "0 6" "0 16"; do
  set -- $cfg
  LR_SUPERSET_DEVICE=$1 LR_SUPERSET_THREADS=$2 python bench.py --cpu-baseline skip --extras off --e2e-steps 1 > gpurun_out/r02bc_$1_$2.log 2>&1
  python - <<XEOF
import json
for l in open("gpurun_out/r02bc_$1_$2.log"):
    if l.startswith("{"):
        d=json.loads(l); print("device=$1 superset_threads=$2", round(d["value"],2), [round(x,1) for x in d["ms_per_job"]], round(d["e2e"]["value"],2), d["job_result"]["vs_reference_run"]["trace_identical"])
XEOF
done
