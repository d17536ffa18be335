#!/bin/bash
# pipelined stream driver: parity tests, then cfg 5 over pipe widths (projection SMs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "pipelined or stream_run" 2>&1 | tail -5
for p in ${PIPES:-0 80 88 92}; do
  timeout 600 python bench.py --config 5 --stream-pipe $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2> gpurun_out/pipe_$p.err | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print('pipe $p', '%.4g' % j['value'], 'ms %.3f' % j['ms_per_step'], j['phases_ms'], j['batch_latency_ms']['p50'], j['batch_latency_ms']['p99'], j['exactness'])
"
  tail -2 gpurun_out/pipe_$p.err
done
