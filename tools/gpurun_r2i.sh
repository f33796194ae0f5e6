python -m pytest tests -q -m gpu -rf -p no:cacheprovider --timeout 1500 > gpurun_out/r2_pytest10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest10.log
