#!/bin/bash
# ncu --set full summaries of the cfg 4 K-streamed kernel and the cfg 5 stream step
# (each only after its own command has run cleanly without ncu)
mkdir -p gpurun_out
python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hash_tck|recheck_segs|convert_x_wide" -s 3 -c 3 \
    -f -o gpurun_out/prof_cfg4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu4.log 2>&1
echo "ncu cfg4 rc=$?"
python bench.py --config 5 --rows 1048576 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_step|hash_tc|convert_x" -s 8 -c 3 \
    -f -o gpurun_out/prof_cfg5 python bench.py --config 5 --rows 1048576 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu5.log 2>&1
echo "ncu cfg5 rc=$?"
