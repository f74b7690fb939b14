# final bench lines of the round, then the ncu launch list and the Cholesky capture of the same build
head -6 tools/round_bench.sh | tail -5 > /tmp/rb.sh; bash /tmp/rb.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_cholesky_tiles -s 3 -c 1 -o gpurun_out/full_k_cholesky_tiles \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chol.log 2>&1; echo chol=$?
