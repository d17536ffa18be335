for d in ${DBGS:-0 16 1 3}; do
  ACE_TC_DBG=$d timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg', $d, round(d['phases_ms']['projection_kernel'],4))"
done
