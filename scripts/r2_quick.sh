#!/bin/bash
# quick check after a kernel change: GPU parity tests, hash timings, section cycles, cfg 2 + cfg 5 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${PYT:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
[ "${PROF:-0}" = 1 ] && bash scripts/r2_hashprof.sh
for c in ${CFGS:-2 5}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', $c, '%.4e'%d['value'], round(d['ms_per_step'],4), d.get('phases_ms'), d.get('batch_latency_ms',{}).get('p50'), d.get('batch_latency_ms',{}).get('p99'))"; done
CFG=5 ROWS=2000000 TAG=q5 bash scripts/launches.sh; cat gpurun_out/launches_q5.txt
SKIP=12 CFG=2 ROWS=500000 TAG=q2 bash scripts/launches.sh; cat gpurun_out/launches_q2.txt
