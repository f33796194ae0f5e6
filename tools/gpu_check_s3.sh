cd $GRAFT_REPO_ROOT
python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 1800 > gpurun_out/pytest_gpu_s3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s3.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s3.txt

tail -3 gpurun_out/pytest_gpu_s3.txt
