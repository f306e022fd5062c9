#!/bin/bash
# gpurun: steps/s and in-step E-pass bandwidth vs look-ahead SMs, repeated
for rep in 1 2; do
for s in 116 140 148; do
  DME_LOOKAHEAD_SMS=$s timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade --steps 100 > gpurun_out/lab_$s.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lab_$s.json')); r=d['roofline']; print('la $s', round(d['value'],1), 'steps/s  epass', round(r['hbm_view']['achieved_gbs']), 'GB/s frac', round(r['frac'],3))"
done; done
