#!/bin/bash
# gpurun: compare in-tree library builds (args: .so names under paper_1805_08990_b200/; "cur" =
# libdme.so): quick bench + ncu launch-list medians of the pipelined step kernels
O=gpurun_out; mkdir -p $O
P=paper_1805_08990_b200
qb() {
timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade > $O/bench_q.json 2> $O/bench_q.err; tail -2 $O/bench_q.err
python -c "
import json
d=json.load(open('gpurun_out/bench_q.json'))
print('steps/s %.1f ms/step %.4f rank %s' % (d['value'], d['ms_per_step'], d['config'].get('rank_after_timed_steps')))"
}
for rep in 1 2; do
for v in "$@"; do
  if [ $v = cur ]; then unset DME_LIB; else export DME_LIB=$PWD/$P/$v; fi
  echo "== $v"; qb
  if [ $rep = 1 ]; then
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_$v.csv python tools/pipe_probe.py > /dev/null 2>&1
    python tools/ll_summary.py $O/ll_$v.csv 200 2>/dev/null | head -12
  fi
done
done
