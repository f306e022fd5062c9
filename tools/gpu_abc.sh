#!/bin/bash
# gpurun: compare library builds / measurement knobs. Args: "cur" (libdme.so), a .so name under
# paper_1805_08990_b200/ (loaded through DME_LIB), or "env:NAME=VALUE" (libdme.so with that knob).
# Quick bench x2 (alternating) + one ncu launch list (kernel medians) per variant.
O=gpurun_out; mkdir -p $O
P=paper_1805_08990_b200
qb() {
timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade > $O/bench_q.json 2> $O/bench_q.err; tail -2 $O/bench_q.err
python -c "
import json
d=json.load(open('gpurun_out/bench_q.json'))
print('steps/s %.1f ms/step %.4f rank %s' % (d['value'], d['ms_per_step'], d['config'].get('rank_after_timed_steps')))"
}
setv() {
  unset DME_LIB; for e in $ENVS; do unset ${e%%=*}; done
  case $1 in
    cur) ;;
    env:*) export ${1#env:}; ENVS="$ENVS ${1#env:}" ;;
    *) export DME_LIB=$PWD/$P/$1 ;;
  esac
}
ENVS=""
for rep in 1 2 3; do
for v in "$@"; do
  setv $v
  echo "== $v"; qb
  if [ $rep = 1 ] && [ -z "$NO_NCU" ]; then
    tag=$(echo $v | tr ':=/' '___')
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ll_$tag.csv python tools/pipe_probe.py > /dev/null 2>&1
    python tools/ll_summary.py $O/ll_$tag.csv 200 2>/dev/null | head -14
  fi
done
done
