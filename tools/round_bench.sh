# plain runs (bench lines + the ncu targets once without ncu)
python bench.py --steps 200 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo cfg3=$?
python bench.py --config cfg2 --steps 200 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo cfg2=$?
python bench.py --config cfg5 --scenes 8 --steps 100 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo cfg5=$?
python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo cfg4=$?
python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for t in pcg emu big; do python tools/ncu_targets.py $t > gpurun_out/plain_$t.log 2>&1; echo $t=$?; done
