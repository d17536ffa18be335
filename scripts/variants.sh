#!/bin/bash
# time alternative builds of libace_dev.so (variants/*.so): SCRIPT (default: bench line of CFG)
cp paper_1706_06664_b200/lib/libace_dev.so /tmp/libace_dev.keep.so
for rep in 1 2; do
for v in variants/*.so; do
  cp $v paper_1706_06664_b200/lib/libace_dev.so
  if [ -n "$SCRIPT" ]; then timeout 300 python $SCRIPT $(basename $v) 2>&1 | tail -1; continue; fi
  timeout 300 python bench.py --config ${CFG:-2} ${ROWS:+--rows $ROWS} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1]); print('$(basename $v)', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d.get('phases_ms',{}).items()})" || tail -3 gpurun_out/var.log
done
done
cp /tmp/libace_dev.keep.so paper_1706_06664_b200/lib/libace_dev.so
