# sparse sweep times vs the fused bottom-subtree height (SPB_SWEEP_FUSE)
for cfg in cfg2 cfg3; do for f in default 2 3 4 5 6 7 8; do
  if [ $f = default ]; then unset SPB_SWEEP_FUSE; else export SPB_SWEEP_FUSE=$f; fi
  timeout 120 python tools/sweep_slots.py $cfg 2>&1 | tail -1 | sed "s/^/$cfg fuse=$f /"
done; done
