# Sensitivity of the cfg4 job to the host's draw throughput: default Omega path vs device assembly, at the
# default thread count and with the draw pool limited (an emulated slower host)
nproc; lscpu | grep -E "Model name|MHz" | head -3
for thr in "" 6 3; do
  for dev in 0 1; do
    LR_HOST_THREADS=$thr LR_SUPERSET_DEVICE=$dev python bench.py --cpu-baseline skip --extras off --e2e-steps 1 > gpurun_out/r02bb_${dev}_t${thr:-all}.log 2>&1
    python - <<XEOF
import json
for l in open("gpurun_out/r02bb_${dev}_t${thr:-all}.log"):
    if l.startswith("{"):
        d=json.loads(l); print("device=$dev threads=${thr:-all}", round(d["value"],2), [round(x,1) for x in d["ms_per_job"]], round(d["e2e"]["value"],2), d["job_result"]["vs_reference_run"]["trace_identical"])
XEOF
  done
done
