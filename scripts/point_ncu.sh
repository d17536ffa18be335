#!/bin/bash
# kernel durations of the per-point loop (ace_point_bench, cfg 5 shapes)
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_1706_06664_b200 import workloads as W
x, _ = W.host_rows(5, 0, 4096 + 200)
x.astype(np.float32).tofile('/tmp/pt_rows.f32')
PY
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${CACHE:-all} -k regex:point --csv --log-file gpurun_out/point_ncu.csv \
  paper_1706_06664_b200/lib/ace_point_bench 64 15 50 1 1.0 4096 0 200 /tmp/pt_rows.f32 > gpurun_out/point_ncu.log 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open('gpurun_out/point_ncu.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
import collections
by = collections.defaultdict(list)
for r in rows[1:]:
    by[r[ki][:40]].append(float(r[vi].replace(',', '')))
for k, v in by.items():
    v.sort()
    print(k, 'launches', len(v), 'median ns', v[len(v) // 2], 'min', v[0], 'max', v[-1])
PY
