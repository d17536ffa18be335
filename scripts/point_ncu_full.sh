#!/bin/bash
# one ncu --set full capture of a per-point kernel (score with a deferred insert)
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_1706_06664_b200 import workloads as W
x, _ = W.host_rows(5, 0, 4096 + 200)
x.astype(np.float32).tofile('/tmp/pt_rows.f32')
PY
ncu --set full --import-source on --clock-control none --cache-control none -k regex:point -s 60 -c 1 \
  -o gpurun_out/point_full -f paper_1706_06664_b200/lib/ace_point_bench 64 15 50 1 1.0 4096 0 200 /tmp/pt_rows.f32 > gpurun_out/point_full.log 2>&1
tail -3 gpurun_out/point_full.log
