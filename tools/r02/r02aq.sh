python -m pytest tests/test_gpu_kernels.py -x -q -k "omega_assembled" 2>&1 | tail -2
for cfg in "1 1" "0 1" "1 1" "0 1"; do
  set -- $cfg
  LR_SUPERSET_DEVICE=$1 LR_OMEGA_SPEC_ESC=$2 python bench.py --cpu-baseline skip --extras off --e2e-steps 1 > gpurun_out/r02aq_$1$2.log 2>&1
  python - <<XEOF
import json
for l in open("gpurun_out/r02aq_$1$2.log"):
    if l.startswith("{"):
        d=json.loads(l); print("device=$1 esc=$2", round(d["value"],2), [round(x,1) for x in d["ms_per_job"]], round(d["e2e"]["value"],2), d["job_result"]["vs_reference_run"]["trace_identical"], "busy", round(sum(k["ms_per_job"] for k in d["roofline_kernels"]),1))
XEOF
done
