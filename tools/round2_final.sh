# Round-2 final evidence on one B200 (run under gpurun from the repo root).
# Plain runs first (bench lines), then the ncu launch list and --set full
# captures; every ncu command line has exited 0 without ncu just before.
set -u
O=gpurun_out
python -m pytest tests -m gpu -q > $O/f_gputest.log 2>&1; echo gputest=$?; tail -2 $O/f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/f_smoke.log 2>&1; echo smoke=$?; tail -1 $O/f_smoke.log
python bench.py --steps 200 --warmup 5 > $O/f_bench_cfg3.json 2> $O/f_bench_cfg3.err; echo cfg3=$?
python bench.py --collider jaw --steps 200 --warmup 5 --no-cpu-baseline > $O/f_bench_cfg3_jaw.json 2> $O/f_bench_cfg3_jaw.err; echo jaw=$?
python bench.py --config cfg2 --steps 300 --warmup 5 > $O/f_bench_cfg2.json 2> $O/f_bench_cfg2.err; echo cfg2=$?
python bench.py --config cfg5 --steps 100 --warmup 5 --no-cpu-baseline > $O/f_bench_cfg5.json 2> $O/f_bench_cfg5.err; echo cfg5=$?
python bench.py --config cfg5 --scenes 8 --steps 100 --warmup 5 > $O/f_bench_cfg5_batch8.json 2> $O/f_bench_cfg5_batch8.err; echo cfg5b=$?
python bench.py --config cfg4 --steps 10 --warmup 3 > $O/f_bench_cfg4.json 2> $O/f_bench_cfg4.err; echo cfg4=$?
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$B > $O/f_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/r02_launches_cfg3.csv $B > $O/f_ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_cholesky_oz -s 2 -c 1 \
  -o $O/r02_full_k_cholesky_oz_cfg3 $B > $O/f_ncu_chol3.log 2>&1; echo chol3=$?
for k in k_dense_backward k_sym_gemv_stream "k_fw_level" k_bw_level k_local_forces k_subtree_forward; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $O/r02_full_$(echo $k | tr -cd 'a-z_') $B > $O/f_ncu_$k.log 2>&1; echo $k=$?
done
B2="python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline"
$B2 > $O/f_plain2.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/r02_launches_cfg2.csv $B2 > $O/f_ncu_launch2.log 2>&1; echo launches2=$?
ncu --set full --clock-control none --import-source on -k regex:k_cholesky -s 2 -c 1 \
  -o $O/r02_full_k_cholesky_cfg2 $B2 > $O/f_ncu_chol2.log 2>&1; echo chol2=$?
