set -x
nproc
python -m pytest tests -q -m gpu -rf -s -p no:cacheprovider --timeout 1200 > gpurun_out/r2_pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest1.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/r2_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2_san_$tool.log
done
