bash tools/ab_build.sh "" "-DTOPT_RDS_TMA_THREADS=128" > gpurun_out/r2_ab13.txt 2>&1
