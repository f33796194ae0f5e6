bash tools/ab_build.sh "" "-DTOPT_RDS_TMA_J1=1" > gpurun_out/r2_ab15.txt 2>&1
