#!/bin/bash
# Round artefacts: full bench line, ncu launch list of the same bench command, and
# ncu --set full captures of the top kernels (each only after its command exited 0 without ncu).
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.log 2>&1 || { tail -20 gpurun_out/bench_full.log; exit 1; }
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
bash tools/prof_multi.sh "k_sl_pipe<.int.0, .bool.1:4" "k_sl_trace2:1" "k_rzmerge:0"
