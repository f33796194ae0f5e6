python -m pytest tests -q -m gpu -rf -p no:cacheprovider --timeout 900 -k "operators or fullsize or derivatives or eval_gradient or linear" > gpurun_out/r2_pytest6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest6.log
bash tools/ab_build.sh "" "-DTOPT_RDS_TMA=0" > gpurun_out/r2_ab6.txt 2>&1
