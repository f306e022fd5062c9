#!/bin/bash
# gpurun: A/B of paper_1805_08990_b200/libdme_old.so (DME_LIB) against the current libdme.so:
# eigen phase probe + quick bench, alternating, twice
O=gpurun_out
mkdir -p $O
qb() {
timeout 300 python bench.py --no-cpu --no-variant --no-e2e --no-sparse --no-pade "$@" > $O/bench_q.json 2> $O/bench_q.err; tail -2 $O/bench_q.err
python - <<'PY'
import json
try:
    d=json.load(open('gpurun_out/bench_q.json')); r=d['roofline']
    print("steps/s %.1f ms/step %.4f rank %s epass frac %.3f eig_share %.2f" % (d['value'], d['ms_per_step'], d['config'].get('rank_after_timed_steps'), r['frac'], r.get('small_eig_share', -1)))
except Exception as e: print("bench parse failed", e)
PY
}
for rep in 1 2; do
  echo "== old"; DME_LIB=$PWD/paper_1805_08990_b200/libdme_old.so timeout 120 python tools/eig_split_probe.py 2>&1 | tail -6
  DME_LIB=$PWD/paper_1805_08990_b200/libdme_old.so qb
  echo "== new"; timeout 120 python tools/eig_split_probe.py 2>&1 | tail -6
  qb
done
