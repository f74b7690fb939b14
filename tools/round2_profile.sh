# Round-2 evidence on one B200 (run under gpurun from the repo root):
# plain bench lines first, then the ncu launch list and one --set full capture
# of the dominant kernel per config (each ncu command preceded by the same
# command exiting 0 without ncu).
set -u
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/p_plain3.json 2> gpurun_out/p_plain3.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_cfg3.csv \
      $B > gpurun_out/p_ncu_launch.log 2>&1; echo launches=$?
$B > gpurun_out/p_plain3b.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_cholesky_oz -s 2 -c 1 \
      -o gpurun_out/r02_full_k_cholesky_oz_cfg3 $B > gpurun_out/p_ncu_chol3.log 2>&1; echo chol3=$?
B2="python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline"
$B2 > gpurun_out/p_plain2.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_cholesky -s 2 -c 1 \
      -o gpurun_out/r02_full_k_cholesky_cfg2 $B2 > gpurun_out/p_ncu_chol2.log 2>&1; echo chol2=$?
