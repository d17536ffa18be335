#!/bin/bash
# one bench line per BASELINE config (device-resident throughput; cfg 2 is the headline line)
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
done
