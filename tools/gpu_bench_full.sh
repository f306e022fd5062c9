#!/bin/bash
# gpurun: build, the default bench line (all variants), the reference arm, ncu launch list
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; tail -3 $O/bench_full.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_full.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant --no-sparse --no-pade > /dev/null 2>&1
cat $O/bench_full.json | head -c 600; echo; cat $O/bench_ref.json | head -c 300
