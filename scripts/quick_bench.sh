#!/bin/bash
# gpu tests + short bench lines for the given configs (default: 2 3)
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for c in ${CFGS:-2 3}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bc_$c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bc_$c.json').read().strip().splitlines()[-1]); print($c, '%.4g' % d['value'], '%.4f ms' % d['ms_per_step'], {k: round(v, 4) for k, v in d['phases_ms'].items()})" || tail -5 gpurun_out/bc_$c.json
done
