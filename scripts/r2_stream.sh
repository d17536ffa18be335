#!/bin/bash
# stream parity tests + cfg 5 bench at several group sizes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYT:+-k "$PYT"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for g in ${GROUPS_:-2 4}; do timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --stream-group $g 2>gpurun_out/bs.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G', $g, '%.4e'%d['value'], round(d['ms_per_step'],3), d.get('phases_ms'), d['batch_latency_ms']['p50'], d['batch_latency_ms']['p99'], d['exactness'])" || tail -5 gpurun_out/bs.err; done
