python -m pytest tests -q -m gpu -p no:cacheprovider -k "operators and (n0 or n4 or 128)" > gpurun_out/r2_pytest17.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest17.log
bash tools/ab_build.sh "" "-DTOPT_RZ_FSTRIDE=0" "-DTOPT_RF_SWZ=0" > gpurun_out/r2_ab17.txt 2>&1
