#!/bin/bash
# per-kernel device times (ncu launch list) of each variants/*.so on cfg 5 (2M-row stream) and cfg 2
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/keep.so
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  for c in ${CFGS:-5 2}; do
    rows=2000000; [ $c = 2 ] && rows=500000; [ $c = 1 ] && rows=100000; export SKIP=200; [ $c != 5 ] && export SKIP=12
    CFG=$c ROWS=$rows TAG=v$c bash scripts/launches.sh
    echo "== $(basename $v) cfg $c"; cat gpurun_out/launches_v$c.txt
  done
done
cp /tmp/keep.so paper_1706_06664_b200/lib/libace_dev.so
