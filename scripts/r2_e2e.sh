#!/bin/bash
# cfg 5 end-to-end (pinned host rows in, flag bitmap out) with and without the pipeline
for p in ${PIPES:-0 88 0 88}; do
  timeout 900 python bench.py --config 5 --stream-pipe $p --steps 3 --warmup 3 --no-cpu-baseline 2> gpurun_out/e2e_$p.err | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print('pipe $p value %.4g' % j['value'], 'e2e %.4g' % j['e2e']['value'], j['clocks'])
"
done
