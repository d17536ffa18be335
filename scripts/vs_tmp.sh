FAST=1 CONFIGS="5" timeout 900 bash scripts/gpu_check.sh 2>&1 | cut -c1-250
timeout 900 python -m pytest tests/test_golden_full_gpu.py -x -q -k stream 2>&1 | tail -2
python scripts/stream_group.py
python scripts/stream_prof.py
