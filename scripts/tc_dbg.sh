#!/bin/bash
# projection-kernel timing under the ACE_TC_DBG experiment switches
for d in ${DBGS:-0 1 3 7}; do
  ACE_TC_DBG=$d timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dbg_$d.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/dbg_$d.log').read().strip().splitlines()[-1]); print('dbg=$d', d['phases_ms'])"
done
