python -m pytest tests/test_gpu_stress.py -q -rf -s -p no:cacheprovider > gpurun_out/r2_pytest_stress.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_stress.log
bash tools/ab_build.sh "" "-DTOPT_SIDE_PRIO=0" > gpurun_out/r2_ab12.txt 2>&1
python __graft_entry__.py > /dev/null 2>&1
bash tools/prof_multi.sh "k_sl_pipe<.int.0, .bool.1:4" "k_sl_trace2:1" "k_rds_tma:1" "k_rzmerge:0" "k_rassemble:0" "k_rdx:1" > gpurun_out/r2_prof_multi.log 2>&1
for i in 1 2 3 4 5 6; do python tools/ncu_summary.py gpurun_out/full_$i.ncu-rep >> gpurun_out/ncu_full_r02_summary.txt 2>&1; done
python tools/ncu_source_summary.py gpurun_out/full_1.ncu-rep 16777216 40 > gpurun_out/ncu_slpipe_r02_source.txt 2>&1
python tools/ncu_source_summary.py gpurun_out/full_2.ncu-rep 16777216 40 > gpurun_out/ncu_trace_r02_source.txt 2>&1
mv gpurun_out/full_1.ncu-rep gpurun_out/r2_full_slpipe.ncu-rep; rm -f gpurun_out/full_*.ncu-rep
