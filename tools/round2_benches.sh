# Round-2 bench lines + GPU suite + smoke on the final build (no ncu; the
# kernels' ncu evidence comes from tools/round2_final.sh).
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
