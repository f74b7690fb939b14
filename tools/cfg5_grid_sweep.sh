# cfg5 batch throughput vs the tile-Cholesky grid per scene (SPB_CHOL_GRID)
for g in 0 12 18 28; do
  if [ $g = 0 ]; then unset SPB_CHOL_GRID; else export SPB_CHOL_GRID=$g; fi
  python bench.py --config cfg5 --scenes 8 --steps 60 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grid', '$g', round(d['value'],1), 'single', round(d['config']['single_scene_ms_per_frame'],3))"
done
