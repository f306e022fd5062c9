#!/bin/bash
for c in 1 2; do for jk in 0 16 24 32 48; do
  DME_JACOBI_K=$jk timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 50 > gpurun_out/jk.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/jk.json')); print('config $c jacobi_k $jk', round(d['value'],1), 'steps/s')"
done; done
