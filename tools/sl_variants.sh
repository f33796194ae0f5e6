#!/bin/bash
# time the SL kernels of the 256^3 bench step for each TOPT_SL_VARIANT
for V in s8 s16 p8 p16; do
  TOPT_SL_VARIANT=$V python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_$V.log 2>&1
  python3 -c "
import json,sys
d=json.loads(open('gpurun_out/var_$V.log').read().strip().splitlines()[-1])
k=d['kernels']
print('$V', d['value'], 'step', k['sl_step']['GB/s'], 'trace', k['sl_trace']['GB/s'], 'last', k['sl_step_last']['GB/s'], 'ef', k['efactor']['GB/s'])"
done
