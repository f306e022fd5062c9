#!/bin/bash
# gpurun iteration: build, GPU tests, short bench, per-kernel launch times of a short bench run
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --no-cpu --no-variant --no-e2e > $O/bench_iter.json 2> $O/bench_iter.err; tail -3 $O/bench_iter.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_iter.json')); r=d['roofline']
print("steps/s %.1f ms/step %.4f  epass %.1f GB/s frac %.3f share %.2f eig_share %.2f gram %.2f apply %.2f prof_ms %.4f" % (d['value'], d['ms_per_step'], r['hbm_view']['achieved_gbs'], r['frac'], r['share_of_step'], r['small_eig_share'], r['gram_share'], r['apply_share'], r['profiled_ms_per_step']))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_iter.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-variant > /dev/null 2>&1
python tools/launch_summary.py $O/launches_iter.csv
