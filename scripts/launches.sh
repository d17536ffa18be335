# launch list (per-kernel device time) of a short cfg run: CFG, ROWS, TAG
CFG=${CFG:-5}; ROWS=${ROWS:-2000000}; TAG=${TAG:-x}
python bench.py --config $CFG --rows $ROWS --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-200} -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --config $CFG --rows $ROWS --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
