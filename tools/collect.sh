#!/bin/bash
# Round artefacts: full bench line, ncu launch list, ncu --set full of the SL step kernel.
set -x
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.log 2>&1
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_sl_tiled<0" -s 12 -c 3 -o gpurun_out/prof_slstep $B > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
