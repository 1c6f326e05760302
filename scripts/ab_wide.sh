#!/bin/bash
# A/B: wide concat kernel (k_concat_wide) vs the generic k_concat (REI_GENERIC_CONCAT=1)
for w in c3-planted-s1-nu c4-planted-s0 c3-big c4-big; do
  for v in wide generic; do
    if [ $v = generic ]; then export REI_GENERIC_CONCAT=1; else unset REI_GENERIC_CONCAT; fi
    echo "== $w $v"
    python scripts/trace_e2e.py $w 3 2>&1 | grep "rep" | tail -2
  done
done
