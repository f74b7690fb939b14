#!/bin/bash
# Sweep the tile-Cholesky claim order on cfg3 (diagnostics): lead, lead growth, partial placement.
out=${1:-gpurun_out/sweep.txt}
for pm in 0 1; do for L in 1 2 3 4; do for D in 8 16 1000; do
  r=$(SPB_CHOL_PMODE=$pm SPB_CHOL_LEAD=$L SPB_CHOL_LDIV=$D timeout 120 python tools/chol_probe.py cfg3 2>&1 | grep "nodeps=0")
  echo "pmode=$pm lead=$L ldiv=$D $r" >> $out
done; done; done
