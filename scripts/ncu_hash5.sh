#!/bin/bash
# ncu --set full + source stall sampling of the projection kernel on a cfg-5-shaped hashing launch
python scripts/tc_prof.py ${CFG:-5} ${ROWS:-262144} > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:hash_tc_kernel -s 5 -c 1 \
  -f -o gpurun_out/prof_${TAG:-h5} python scripts/tc_prof.py ${CFG:-5} ${ROWS:-262144} > gpurun_out/ncu_${TAG:-h5}.log 2>&1
