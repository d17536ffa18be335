# GPU check: parity suites (fast, then full-size unless FAST=1) + one bench line per config
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -15
[ -z "$FAST" ] && timeout 2400 python -m pytest tests -x -q -m "gpu and slow" 2>&1 | tail -15
for c in ${CONFIGS:-2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-900
done
