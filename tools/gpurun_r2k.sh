python -m pytest tests/test_gpu_stress.py -q -rf -s -p no:cacheprovider > gpurun_out/r2_pytest_stress.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_stress.log
bash tools/prof_multi.sh "k_sl_pipe<.int.0, .bool.1:4" "k_sl_trace2:1" "k_rds_tma:1" "k_rzmerge:0" "k_rassemble:0" "k_rdx:1" > gpurun_out/r2_prof_multi.log 2>&1
