#!/bin/bash
# A/B: bench the 256^3 step for each set of extra nvcc flags given as arguments ("" = default)
for X in "$@"; do
  TOPT_NVCC_EXTRA="$X" python __graft_entry__.py > gpurun_out/build_ab.log 2>&1 || { echo "build failed: $X"; tail -5 gpurun_out/build_ab.log; continue; }
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab.log 2>&1
  python3 -c "
import json
d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('[$X]', d['value'], {k: v['GB/s'] for k, v in d['kernels'].items()})"
done
