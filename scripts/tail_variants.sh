#!/bin/bash
# detect-tail phase timeline (scripts/tail_prof.py) for each variants/*.so
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/libace_dev.keep.so
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  echo "$(basename $v): $(python scripts/tail_prof.py ${CFGS:-2} 2>&1 | tr '\n' ' ')"
done
cp /tmp/libace_dev.keep.so paper_1706_06664_b200/lib/libace_dev.so
