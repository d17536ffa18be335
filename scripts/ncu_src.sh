# ncu source-level stall sampling of the projection kernel: CFG ROWS TAG
CFG=${CFG:-5}; ROWS=${ROWS:-131072}; TAG=${TAG:-src}
python scripts/tc_prof.py $CFG $ROWS > gpurun_out/src_plain.log 2>&1 &&
ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section InstructionStats --clock-control none --import-source on --warp-sampling-interval 0 -k regex:hash_tc_kernel -s 5 -c 1 -o gpurun_out/prof_$TAG -f python scripts/tc_prof.py $CFG $ROWS > gpurun_out/ncu_$TAG.log 2>&1
