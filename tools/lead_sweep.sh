out=gpurun_out/sweep2.txt; : > $out
for L in 1 2 3 4; do for D in 8 16 1000; do
  r=$(SPB_CHOL_LEAD=$L SPB_CHOL_LDIV=$D timeout 120 python tools/chol_probe.py cfg3 2>&1 | grep " ms ")
  echo "lead=$L ldiv=$D $r" >> $out
done; done
