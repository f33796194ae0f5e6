python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "operators or fullsize or parity" > gpurun_out/r2_pytest20.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest20.log
bash tools/ab_build.sh "" "-DTOPT_SL_QUAD=0" > gpurun_out/r2_ab20.txt 2>&1
