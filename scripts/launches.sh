#!/bin/bash
# per-kernel device times of a short bench run (ncu launch list), summarised
#   scripts/launches.sh OUT.csv [extra bench.py args]
OUT=${1:-gpurun_out/launches.csv}
shift
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_launch.log 2>&1
python scripts/summarize_launches.py $OUT
