#!/bin/bash
# Sweep (G,T) for the cfg4 widths (tools/spmm_cfg4_probe.py) -- experiments only.
for gt in default 2,3 2,4 4,2 4,3 4,4 8,2 8,3 16,2; do
  if [ $gt = default ]; then python tools/spmm_cfg4_probe.py | sed "s/^/$gt /"; else LR_SPMM_GT=$gt python tools/spmm_cfg4_probe.py | sed "s/^/$gt /"; fi
done
