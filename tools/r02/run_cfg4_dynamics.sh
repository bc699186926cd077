#!/bin/bash
# one process per setting, each under its own timeout
out=${1:-gpurun_out/r02_cfg4_dynamics.txt}
: > $out
for c in ${CFGS:-"10:1.0:0.17:60" "1:1.0:0.17:60" "1:0.5:0.17:60" "0:0:0.3:30" "40:1.0:0.3:80" "10:1.9:0.25:80"}; do
  CFG=$c timeout ${TMO:-150} python tools/r02/cfg4_dynamics.py >> $out 2>&1 || echo "timeout/exit $? for $c" >> $out
done
