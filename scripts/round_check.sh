#!/bin/bash
# GPU round check: tests, bench (both arms), launch list, ncu --set full of the top kernel
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  ./scripts/launches.sh gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"hash_tc|convert_x|detect_tail" -s 6 -c 3 \
      -f -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
