set -e
python scripts/stream_prof.py > gpurun_out/sp_plain.log 2>&1
cat gpurun_out/sp_plain.log
ncu --set full --clock-control none --import-source on -k regex:stream_apply -s 40 -c 2 -o gpurun_out/prof_sa -f python scripts/stream_prof.py > gpurun_out/ncu_sa.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hash_tc_kernel -s 30 -c 1 -o gpurun_out/prof_h64 -f python scripts/stream_prof.py > gpurun_out/ncu_h64.log 2>&1
