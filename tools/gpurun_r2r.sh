python -m pytest tests -q -m gpu -p no:cacheprovider -rf -k "operators or fullsize or parity or slabs or solve_native or linear or edge or flowmap" > gpurun_out/r2_pytest21.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest21.log
bash tools/ab_build.sh "" "-DTOPT_RS_TMA=0" > gpurun_out/r2_ab21.txt 2>&1
