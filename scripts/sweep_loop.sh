#!/bin/bash
# time-to-minimal-RE vs the device level loop's level-size limit (REI_DEVICE_LOOP_CAND)
for w in table1-row1 table1-row8 c2-t1-s0; do
  for c in 0 4194304 16777216 67108864; do
    if [ "$c" = 0 ]; then export REI_NO_DEVICE_LOOP=1; else unset REI_NO_DEVICE_LOOP; export REI_DEVICE_LOOP_CAND=$c; fi
    echo "== $w cand_limit=$c"
    REI_TRACE=1 python scripts/trace_e2e.py $w 5 2>&1 | grep "rep\|device loop" | tail -4
  done
done
