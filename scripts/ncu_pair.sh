#!/bin/bash
# ncu --set full + source sampling of the stream kernel (cfg 5, 2M-row stream)
python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pp_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:stream_solo -s 10 -c 1 \
  -f -o gpurun_out/prof_${TAG:-pair} python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pair.log 2>&1
