# quick GPU check: parity suite + one bench line per config (builder runs)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -15
for c in ${CONFIGS:-2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -3
done
