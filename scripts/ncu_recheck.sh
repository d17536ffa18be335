python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rn_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:recheck_near -s 8 -c 1 -f -o gpurun_out/prof_rn python bench.py --config 5 --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rn.log 2>&1
