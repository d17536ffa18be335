#!/bin/bash
# per-point kernel duration (ncu, warm) and loop rate for each variants/*.so
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/libace_dev.keep.so
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  echo "== $v $(CACHE=none bash scripts/point_ncu.sh 2>&1 | tail -1)"
  paper_1706_06664_b200/lib/ace_point_bench 64 15 50 1 1.0 4096 200 /tmp/pt_rows.f32
done
cp /tmp/libace_dev.keep.so paper_1706_06664_b200/lib/libace_dev.so
