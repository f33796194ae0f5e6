#!/bin/bash
# Quick ncu metrics for kernels matching a demangled-name regex in a short bench run.
# usage: bash tools/ncu_quick.sh "<regex>" <count> <out-name> [bench args]
K=$1; C=${2:-3}; O=${3:-quick}; shift 3
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__occupancy_limit_shared_mem,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e $@"
$B > gpurun_out/plain_$O.log 2>&1 || { tail -5 gpurun_out/plain_$O.log; exit 1; }
ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:$K" -c $C --csv --log-file gpurun_out/ncu_$O.csv $B > gpurun_out/ncu_$O.out 2> gpurun_out/ncu_$O.err
python3 tools/ncu_quick_print.py gpurun_out/ncu_$O.csv
