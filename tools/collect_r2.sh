#!/bin/bash
# Round-2 artefacts: the default bench line, the other configs' lines, the replica sweeps, and the
# ncu launch list of the bench command (run after it exited 0 without ncu).
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r02.log 2>&1 && tail -1 gpurun_out/bench_r02.log > gpurun_out/bench_r02.json
python bench.py --config 1 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_r02_config1.log 2>&1
python bench.py --config 2 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_r02_config2.log 2>&1
python bench.py --config 3 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_r02_config3.log 2>&1
python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r02_config5.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02_reference.log 2>&1
bash tools/run_sweeps.sh
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch_r02.log 2>&1
echo done
