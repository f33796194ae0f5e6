B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --solver-iters 0"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_sl_quad<.bool.1" -s 4 -c 1 -o gpurun_out/r2_quad $B > gpurun_out/r2_ncu_quad.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_quad.ncu-rep > gpurun_out/r2_quad_summary.txt 2>&1
python tools/ncu_source_summary.py gpurun_out/r2_quad.ncu-rep 16777216 50 > gpurun_out/r2_quad_source.txt 2>&1
