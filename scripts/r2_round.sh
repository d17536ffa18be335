#!/bin/bash
# round-2 check: tests, smoke, bench (all configs, both arms, point API), launch lists, ncu captures
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --api point > gpurun_out/bench_point.json 2> gpurun_out/bench_point.err; echo "point rc=$?"
if [ "${NCU:-1}" = "1" ]; then
  SKIP=20 CFG=5 ROWS=4000000 TAG=r5 bash scripts/launches.sh; cat gpurun_out/launches_r5.txt
  SKIP=12 CFG=2 ROWS=500000 TAG=r2 bash scripts/launches.sh; cat gpurun_out/launches_r2.txt
  ROWS=524288 TAG=h5 bash scripts/ncu_hash5.sh; echo "ncu h5 rc=$?"
  CFG=2 ROWS=500000 TAG=h2 bash scripts/ncu_hash5.sh; echo "ncu h2 rc=$?"
  TAG=pair bash scripts/ncu_pair.sh; echo "ncu pair rc=$?"
fi
