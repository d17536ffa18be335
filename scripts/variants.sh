#!/bin/bash
# time alternative builds of libace_dev.so (variants/*.so) with the bench
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  timeout 120 python scripts/tc_quick.py 2>&1 | grep -c "mismatches=0" | sed "s/^/$(basename $v) exact_cases=/"
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1]); print('$(basename $v)', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phases_ms'].items()})"
done
