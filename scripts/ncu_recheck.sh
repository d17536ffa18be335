#!/bin/bash
# ncu --set full + source sampling of the near-tie kernel (CFG, default 2)
CFG=${CFG:-2}
python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rn_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:recheck_near -s 3 -c 1 -f -o gpurun_out/prof_rn \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rn.log 2>&1
