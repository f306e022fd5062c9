#!/bin/bash
# gpurun: compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the small workload
O=gpurun_out/sanitizer
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  for part in dense sparse; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --log-file $O/${tool}_${part}.log python tools/sanitize_workload.py $part > $O/${tool}_${part}.out 2>&1
    echo "$tool $part rc=$? $(grep -c 'ERROR SUMMARY\|RACECHECK SUMMARY' $O/${tool}_${part}.log) $(grep 'SUMMARY' $O/${tool}_${part}.log | tail -1)"
  done
done
