#!/bin/bash
# projection-kernel section cycles (ACE_TC_PROF build in variants/prof.so) and plain timings
mkdir -p gpurun_out
python scripts/hash_time.py lib > gpurun_out/hash_time.txt 2>&1
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/keep.so
cp variants/prof.so paper_1706_06664_b200/lib/libace_dev.so
for a in "5 524288" "2" "3 2000000"; do python scripts/tc_prof.py $a; done > gpurun_out/tc_prof.txt 2>&1
cp /tmp/keep.so paper_1706_06664_b200/lib/libace_dev.so
cat gpurun_out/hash_time.txt gpurun_out/tc_prof.txt
