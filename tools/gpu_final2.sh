#!/bin/bash
# Final evidence after the sparse-A path: build, all GPU tests, smoke, default bench, ncu of one
# sparse E_h action (config 5, k = 46).
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench5.json 2> $O/bench5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cheb_reg_kernel -c 1 -o $O/cheb_one -f python tools/cheb_one.py 46 > $O/ncu_cheb.log 2>&1
ncu -i $O/cheb_one.ncu-rep --page details > $O/cheb_details.txt 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; python -c "
import json; d=json.load(open('gpurun_out/bench5.json')); print(d['value'], d['time_to_T_s'], d['roofline']['frac']); print(json.dumps(d['sparse_variant']))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant --no-sparse > /dev/null 2>&1
python tools/launch_summary.py $O/launches_final.csv > $O/launches_summary.txt 2>&1; tail -3 $O/launches_summary.txt
