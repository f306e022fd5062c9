#!/bin/bash
# gpurun: racecheck + initcheck re-run after fixes; sturm microbenchmark
O=gpurun_out/sanitizer
mkdir -p $O
for tool in racecheck initcheck memcheck synccheck; do
  for part in dense sparse; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --log-file $O/${tool}_${part}.log python tools/sanitize_workload.py $part > $O/${tool}_${part}.out 2>&1
    echo "$tool $part rc=$? $(grep 'SUMMARY' $O/${tool}_${part}.log | tail -1)"
  done
done
./tools/sturm_probe
