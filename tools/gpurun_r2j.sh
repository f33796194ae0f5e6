python scratch/diag_stress.py > gpurun_out/r2_diag_stress.txt 2>&1
