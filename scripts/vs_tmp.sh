FAST=1 CONFIGS="5 2 3 1" bash scripts/gpu_check.sh 2>&1 | cut -c1-330
cp variants/prof.so paper_1706_06664_b200/lib/libace_dev.so
python scripts/tc_prof.py 5 131072; python scripts/tc_prof.py 2
