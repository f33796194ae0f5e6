python -m pytest tests -q -m gpu -rf -s -p no:cacheprovider --timeout 1500 > gpurun_out/r2_pytest4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest4.log
bash tools/ab_build.sh "" "-DTOPT_SL_TMA=0" > gpurun_out/r2_ab4.txt 2>&1
