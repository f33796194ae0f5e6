python -m pytest tests -q -m gpu -rf -s -p no:cacheprovider --timeout 900 -k "linear or solve_native or slabs" > gpurun_out/r2_pytest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest3.log
python bench.py --steps 30 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo "bench rc=$?" >> gpurun_out/r2_bench3.err
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --solver-iters 0"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_sl_pipe<.int.0, .bool.1" -s 4 -c 1 -o gpurun_out/r2_slpipe $B > gpurun_out/r2_ncu_slpipe.log 2>&1
tail -2 gpurun_out/r2_ncu_slpipe.log
