#!/bin/bash
# Round-2 artefacts of the final tree: the default bench line, the other configs' lines, the
# reference arm, the ncu launch list of the bench command (run after it exited 0 without ncu), ncu
# --set full captures of the top kernels summarised here (the .ncu-rep files are too large to bring
# back), the whole -m gpu suite and the smoke.  (Replica sweeps: tools/run_sweeps.sh.)
python __graft_entry__.py > gpurun_out/build_r02.log 2>&1 || { echo build failed; exit 1; }
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r02.log 2>&1 && tail -1 gpurun_out/bench_r02.log > gpurun_out/bench_r02.json
python bench.py --config 1 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_r02_config1.log 2>&1
python bench.py --config 2 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_r02_config2.log 2>&1
python bench.py --config 3 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_r02_config3.log 2>&1
python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r02_config5.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02_reference.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch_r02.log 2>&1
bash tools/prof_multi.sh "k_sl_pipe<.int.0, .bool.1:4" "k_sl_trace2:1" "k_rds_tma:1" "k_rzmerge:0" "k_rassemble:0" "k_rstrided_tma:0" > gpurun_out/prof_multi_r02.log 2>&1
rm -f gpurun_out/ncu_full_r02_summary.txt
for i in 1 2 3 4 5 6; do python tools/ncu_summary.py gpurun_out/full_$i.ncu-rep >> gpurun_out/ncu_full_r02_summary.txt 2>&1; done
python tools/ncu_source_summary.py gpurun_out/full_1.ncu-rep 16777216 40 > gpurun_out/ncu_slpipe_r02_source.txt 2>&1
python tools/ncu_source_summary.py gpurun_out/full_2.ncu-rep 16777216 40 > gpurun_out/ncu_trace_r02_source.txt 2>&1
python tools/ncu_traffic.py gpurun_out/full_1.ncu-rep sl_step k_sl_pipe 256 256 256 > gpurun_out/ncu_traffic.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
rm -f gpurun_out/full_*.ncu-rep
bash tools/gpu_tests_r2.sh
echo done
