#!/bin/bash
# gpurun: full-size parity of configs 1-4 and one bench line per config
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1800 python -m pytest -x -q -m gpu tests/test_gpu_configs.py 2>&1 | tail -6
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c --no-sparse --no-pade --no-variant > $O/bench_c$c.json 2> $O/bench_c$c.err
  python -c "import json; d=json.load(open('$O/bench_c$c.json')); print('config $c', round(d['value'],1), 'steps/s', 'ttT', round(d['time_to_T_s'],4), 'rank', d['config']['rank_after_timed_steps'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))" || tail -3 $O/bench_c$c.err
done
