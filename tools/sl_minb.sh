#!/bin/bash
# bench the 256^3 step for SL register budgets (resident blocks per SM 3 and 2)
for B in 2 3; do
  TOPT_NVCC_EXTRA="-DTOPT_SL_MINB=$B" python __graft_entry__.py > gpurun_out/build_$B.log 2>&1
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/minb_$B.log 2>&1
  python3 -c "
import json
d=json.loads(open('gpurun_out/minb_$B.log').read().strip().splitlines()[-1])
print('minb $B', d['value'], {k: v['GB/s'] for k, v in d['kernels'].items()})"
done
