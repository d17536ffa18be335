# ncu --set full of the projection kernel on cfg 2 (and the cfg 5 stream), after plain runs
set -e
python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_plain2.log 2>&1
python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 > gpurun_out/ncu_plain5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hash_tc_kernel -s 4 -c 1 -o gpurun_out/prof_hash_cfg2 -f \
  python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hash_tc_kernel|stream_step" -s 20 -c 2 -o gpurun_out/prof_cfg5 -f \
  python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 > gpurun_out/ncu5.log 2>&1
