#!/bin/bash
# Sweep rows per CTA of the tridiagonalization (LR_TD_ROWS) at the BKI widths.
for r in 4 8 12 16 24; do
  LR_TD_ROWS=$r LR_SYEVD_TIMING=1 python tools/eig_probe.py 2>&1 | grep -E "^syevd n=(260|660|1300) G" | head -3 | sed "s/^/rows=$r /"
done
