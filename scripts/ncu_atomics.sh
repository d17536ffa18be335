#!/bin/bash
# insertion evidence: shared-memory atomics, their bank conflicts and the L2 RED
# merges of the detect tail (cfg 2) and the stream step (cfg 5)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed_op_shared_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_atom.sum
python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"detect_tail" -s 3 -c 1 --csv \
    python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/atom_cfg2.csv 2>gpurun_out/atom_cfg2.err
echo "cfg2 rc=$?"
ncu --metrics $M --clock-control none -k regex:"stream_step" -s 20 -c 1 --csv \
    python bench.py --config 5 --rows 2097152 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/atom_cfg5.csv 2>gpurun_out/atom_cfg5.err
echo "cfg5 rc=$?"
