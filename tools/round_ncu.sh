# ncu evidence (run only after tools/round_bench.sh exited 0 on the same build)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/full_k_pcg \
    python tools/ncu_targets.py pcg > gpurun_out/ncu_pcg.log 2>&1; echo pcg=$?
ncu --set full --clock-control none --import-source on -k regex:k_cholesky_ranks -c 1 -o gpurun_out/full_k_cholesky_ranks \
    python tools/ncu_targets.py emu > gpurun_out/ncu_emu.log 2>&1; echo emu=$?
ncu --set full --clock-control none --import-source on -k regex:k_cholesky_tiles -c 1 -o gpurun_out/full_k_cholesky_tiles_m12288 \
    python tools/ncu_targets.py big > gpurun_out/ncu_big.log 2>&1; echo big=$?
