#!/bin/bash
# gpurun: quick bench A/B for configs 1, 2, 5 (args as tools/gpu_abc.sh: cur / lib.so / env:K=V)
P=paper_1805_08990_b200
for c in ${CFGS:-1 2 5}; do
for rep in 1 2; do
for v in "$@"; do
  for e in $(env | grep -o '^DME_[A-Z_0-9]*'); do unset $e; done
  case $v in cur) ;; env:*) export ${v#env:} ;; *) export DME_LIB=$PWD/$P/$v ;; esac
  timeout 300 python bench.py --config $c --no-cpu --no-variant --no-e2e --no-sparse --no-pade > gpurun_out/q.json 2> gpurun_out/q.err
  python -c "
import json; d=json.load(open('gpurun_out/q.json')); print('config $c $v steps/s %.1f ms/step %.4f' % (d['value'], d['ms_per_step']))" || tail -2 gpurun_out/q.err
done; done; done
