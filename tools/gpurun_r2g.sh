python -m pytest tests -q -m gpu -rf -s -p no:cacheprovider --timeout 1500 > gpurun_out/r2_pytest7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest7.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke7.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke7.log
