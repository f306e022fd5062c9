#!/bin/bash
# gpurun: steps/s of the default bench config vs the look-ahead stream's CTA count
for s in ${@:-140 120 100 80}; do
  DME_LOOKAHEAD_SMS=$s timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade --steps 50 > gpurun_out/la_$s.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/la_$s.json')); print('la $s', round(d['value'],1), 'steps/s', d['config'].get('rank_after_timed_steps'))"
done
