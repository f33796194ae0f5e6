# final-tree GPU test run: the whole -m gpu suite and the smoke
python -m pytest tests -q -m gpu -rA -p no:cacheprovider --timeout 1800 > gpurun_out/pytest_gpu_r02.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/pytest_gpu_r02.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/pytest_gpu_r02.txt
