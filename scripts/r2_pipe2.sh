#!/bin/bash
# pipelined stream driver: cfg 5 over (group, pipe) pairs: "G:P G:P ..."
mkdir -p gpurun_out
for gp in ${GPS:-8:88 16:88 16:92 4:88}; do
  g=${gp%%:*}; p=${gp##*:}
  timeout 600 python bench.py --config 5 --stream-group $g --stream-pipe $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2> gpurun_out/pipe_$g_$p.err | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print('G $g pipe $p', '%.4g' % j['value'], 'ms %.3f' % j['ms_per_step'], j['phases_ms'], 'p50 %.3f p99 %.3f' % (j['batch_latency_ms']['p50'], j['batch_latency_ms']['p99']), j['exactness']['reported'])
"
done
