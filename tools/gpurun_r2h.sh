python -m pytest tests -q -m gpu -rf -p no:cacheprovider --timeout 900 -k "operators or parity or fullsize or slabs or edge" > gpurun_out/r2_pytest9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest9.log
bash tools/ab_build.sh "" "-DTOPT_TRACE_MINB=3" "-DTOPT_RDS_TMA_J1=0" > gpurun_out/r2_ab9.txt 2>&1
