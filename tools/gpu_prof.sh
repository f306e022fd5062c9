#!/bin/bash
# gpurun: build, ncu launch list of a short bench run, per-kernel summary of one step
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_p.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-variant --no-sparse > /dev/null 2>&1
python tools/launch_summary.py $O/launches_p.csv | tail -${1:-40}
