#!/bin/bash
# ncu --set full of the top kernels of the 256^3 bench step (one launch each).
# usage: bash tools/prof_multi.sh "<demangled-name regex>:<skip>" ...
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 || exit 1
i=0
for KS in "$@"; do
  i=$((i+1))
  K="${KS%:*}"; S="${KS##*:}"
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${K}" -s $S -c 1 \
      -o gpurun_out/full_$i $B > gpurun_out/ncu_full_$i.log 2>&1
  tail -1 gpurun_out/ncu_full_$i.log
done
