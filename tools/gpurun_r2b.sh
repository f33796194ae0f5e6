# round-2 GPU check: new parity / slab / native-solve tests, smoke, a short bench
python -m pytest tests -q -m gpu -rf -s -p no:cacheprovider --timeout 1500 -k "operators or parity or slabs or edge or solve_native or host or solver" > gpurun_out/r2_pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?" >> gpurun_out/r2_bench2.err
