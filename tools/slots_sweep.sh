# forward level-kernel variant x slot sizing (one process per setting)
for v in 0 1 2; do for fw in 2 3 4 6; do
  SPB_FW_VARIANT=$v SPB_FW_SLOTS=$fw timeout 120 python tools/sweep_slots.py cfg3 2>&1 | tail -1 | sed "s/^/variant=$v /"
done; done
