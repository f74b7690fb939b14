# Forward level plan sweep (diagnostics; needs an SPB_FW_PLAN="level:R:variant" override in sparse.cu,
# not in the tree): the whole forward sweep time with one level's (R, variant) overridden.
cfg=${1:-cfg3}
t() { SPB_FW_AUTO=0 SPB_FW_PLAN="$1" timeout 200 python tools/kernel_times.py $cfg 2>/dev/null | tr '|' '\n' | grep -o "sparse_forward [0-9.]*" | cut -d' ' -f2; }
echo "base $(t '') $(t '') $(t '')"
for l in 6 7 8 9 10 11 12 13 14 15; do
  line="L$l:"
  for c in 8:0 16:0 32:0 16:2 32:2 64:2 128:2 32:1; do
    R=${c%%:*}; V=${c##*:}
    line="$line $c=$(t "$l:$R:$V")"
  done
  echo "$line"
done
