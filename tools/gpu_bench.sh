#!/bin/bash
# gpurun: build, bench (default), bench reference arm, ncu launch list of a short bench run
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > $O/bench_ncu.log 2>&1
cat $O/bench.json
