#!/bin/bash
# NEXT-3 replica sweeps on one GPU: the paper's alpha grid at 256^2 with
# n_t = 4 and the mesh ladder 64^2 .. 512^2, n_t = 4 .. 32, eps_rel = 1e-3; the w x (sigma, tau)
# grid at 256^2.  Tables land in gpurun_out/, JSON rows beside them.
python sweep.py --grid alpha --n 256 --nt 4 --max-iter 200 --eps 5e-2 --json gpurun_out/sweep_alpha_256.jsonl > gpurun_out/sweep_alpha_256.txt 2>&1
python sweep.py --grid mesh --max-iter 200 --eps 1e-3 --json gpurun_out/sweep_mesh.jsonl > gpurun_out/sweep_mesh.txt 2>&1
python sweep.py --grid wst --n 256 --nt 4 --alpha 1e-2 --max-iter 200 --eps 5e-2 --json gpurun_out/sweep_wst_256.jsonl > gpurun_out/sweep_wst_256.txt 2>&1
