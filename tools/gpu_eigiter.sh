#!/bin/bash
# gpurun: build, selected GPU tests, eigen phase probe, timeline, quick bench; args: pytest selectors
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest -x -q -m gpu "${@:-tests}" 2>&1 | tail -8
timeout 120 python tools/eig_split_probe.py 2>&1 | tail -8
DME_TIMELINE=1 timeout 120 python tools/timeline.py > $O/timeline.log 2>&1; tail -40 $O/timeline.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade > $O/bench_q.json 2> $O/bench_q.err; tail -3 $O/bench_q.err
python - <<'PY'
import json
try:
    d=json.load(open('gpurun_out/bench_q.json')); r=d['roofline']
    print("steps/s %.1f ms/step %.4f rank %s epass frac %.3f eig_share %.2f" % (d['value'], d['ms_per_step'], d['config'].get('rank_after_timed_steps'), r['frac'], r.get('small_eig_share', -1)))
except Exception as e: print("bench parse failed", e)
PY
done
