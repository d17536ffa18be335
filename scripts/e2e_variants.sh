#!/bin/bash
# e2e (C-ABI call with pinned host rows) of each variants/*.so
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/libace_dev.keep.so
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  echo "$(basename $v): $(python scripts/e2e_chunks.py ${CFG:-2} 2>&1 | tail -1)"
done
cp /tmp/libace_dev.keep.so paper_1706_06664_b200/lib/libace_dev.so
