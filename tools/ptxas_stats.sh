#!/bin/bash
# usage: tools/ptxas_stats.sh <file.cu> [grep-regex]   -> kernel, registers, spills, stack
F=$1; R=${2:-.}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -v -c $F -o /tmp/ptxas_stats.o 2>&1 | awk '
/Compiling entry function/ {name=$0; sub(/.*function .?/,"",name); sub(/.? for .*/,"",name)}
/stack frame/ {stack=$5; spst=$9; spld=$13}
/Used [0-9]+ registers/ {for(i=1;i<=NF;i++) if($i=="Used") regs=$(i+1); cmd="c++filt " name; cmd | getline dn; close(cmd); printf "%4d regs  stack %4s  spill %s/%s  %s\n", regs, stack, spst, spld, dn}
/error/ {print}' | grep -E "$R"
