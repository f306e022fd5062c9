#!/bin/bash
# gpurun: end-of-session evidence: all GPU tests, smoke, sanitizer (dense workload), full bench line
O=gpurun_out
mkdir -p $O/sanitizer
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --log-file $O/sanitizer/${tool}_dense.log python tools/sanitize_workload.py dense > $O/sanitizer/${tool}_dense.out 2>&1
  echo "$tool dense rc=$? $(grep 'SUMMARY' $O/sanitizer/${tool}_dense.log | tail -1)"
done
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err; tail -2 $O/bench_final.err
python -c "
import json; d=json.load(open('$O/bench_final.json'))
print('steps/s %.1f ms %.4f ttT %.4f e2e %.1f frac %.3f rank %s clocks %s' % (d['value'], d['ms_per_step'], d['time_to_T_s'], d['e2e']['value'], d['roofline']['frac'], d['config']['rank_after_timed_steps'], d['clocks']))"
