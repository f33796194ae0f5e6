#!/bin/bash
# usage: bash tools/prof.sh <kernel regex> <skip> <count> <outname> [bench args...]
K=${1:-k_sl_tiled}; S=${2:-12}; C=${3:-2}; O=${4:-prof}; shift 4
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e $@"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/$O $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
