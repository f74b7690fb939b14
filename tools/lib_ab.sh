# A/B of two in-tree library builds on cfg3, alternated (diagnostics): bash tools/lib_ab.sh <libA> <libB> <rounds>
out=gpurun_out/lib_ab.txt; : > $out
for r in $(seq 1 ${3:-3}); do for L in $1 $2; do
  SPB_LIB_NAME=$L timeout 200 python bench.py --steps 200 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value'],2), round(d['phases_ms']['local_alpha+forces']*1e3,1))" >> $out
done; done
