#!/bin/bash
# section cycles of the projection kernel for each variants/*.so (ACE_TC_PROF builds)
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/keep.so
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  echo "== $(basename $v)"
  for a in ${ARGS:-"5 262144" "2"}; do python scripts/tc_prof.py $a 2>&1 | grep -E "cfg|mma wait|mma loop|kernel total|epi|pack|conv pass"; done
done
cp /tmp/keep.so paper_1706_06664_b200/lib/libace_dev.so
