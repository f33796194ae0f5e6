python scratch/diag_solve.py c4_64_a1e-03_w3 c4_64_a1e-03_w10 > gpurun_out/r2_diag_solve.txt 2>&1
bash tools/ab_build.sh "-DTOPT_SL_TMA=0" "-DTOPT_SL_TMA=0 -DTOPT_RDS_TMA=0" > gpurun_out/r2_ab5.txt 2>&1
