# Marginal cost of every upper level in the PDL-chained sweeps (diagnostics):
# sweep time with all levels, without each level, without each level's gather.
cfg=${1:-cfg3}
run() { timeout 200 python tools/kernel_times.py $cfg 2>/dev/null | tr '|' '\n' | grep -E "sparse_(forward|backward)" | tr '\n' ' '; echo; }
echo "all: $(run)"
for l in 6 7 8 9 10 11 12 13 14 15; do
  m=$((1 << l))
  echo "skip $l: $(SPB_SWEEP_SKIP=$m run)   gather-only skip: $(SPB_SWEEP_SKIPG=$m run | grep -o 'sparse_forward [0-9.]* us')"
done
echo "skip all gathers: $(SPB_SWEEP_SKIPG=0xffff0 run)"
