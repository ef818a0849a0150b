#!/bin/bash
# Per-kernel pipe mix of one frame (run under gpurun):  tools/pipes.sh [config] OUT.csv
C=${1:-5}; OUT=${2:-gpurun_out/pipes.csv}
python tools/one_frame.py $C > gpurun_out/one_frame.log 2>&1 && \
ncu --profile-from-start off --clock-control none --csv --log-file $OUT --metrics \
gpu__time_duration.sum,sm__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_uniform.sum,sm__inst_executed_pipe_adu.sum,sm__inst_executed_pipe_cbu.sum,sm__inst_executed_pipe_xu.sum,sm__pipe_alu_cycles_active.sum,sm__pipe_fma_cycles_active.sum,sm__pipe_fp64_cycles_active.sum,sm__cycles_elapsed.avg \
python tools/one_frame.py $C
