#!/bin/bash
# gpurun: A/B (libdme_old.so via DME_LIB vs libdme.so): isolated + pipelined eigen phase probes,
# ncu launch list of the step kernels (durations), quick bench
O=gpurun_out
mkdir -p $O
qb() {
timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade "$@" > $O/bench_q.json 2> $O/bench_q.err; tail -2 $O/bench_q.err
python -c "
import json
d=json.load(open('gpurun_out/bench_q.json')); r=d['roofline']
print('steps/s %.1f ms/step %.4f rank %s' % (d['value'], d['ms_per_step'], d['config'].get('rank_after_timed_steps')))"
}
for v in old new; do
  if [ $v = old ]; then export DME_LIB=$PWD/paper_1805_08990_b200/libdme_old.so; else unset DME_LIB; fi
  echo "== $v"
  timeout 120 python tools/eig_split_probe.py 2>&1 | tail -6
  timeout 120 python tools/pipe_probe.py 2>&1 | tail -3
  qb
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_$v.csv python tools/pipe_probe.py > /dev/null 2>&1
  python tools/ll_summary.py $O/ll_$v.csv 200
done
