cp paper_1706_06664_b200/lib/libace_dev.so /tmp/keep.so
for v in variants/*.so; do cp $v paper_1706_06664_b200/lib/libace_dev.so; echo "== $v"; timeout 200 python scripts/skew_bench.py; done
cp /tmp/keep.so paper_1706_06664_b200/lib/libace_dev.so
