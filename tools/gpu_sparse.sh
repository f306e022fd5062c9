O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -25
timeout 300 python bench.py --no-cpu --no-variant --no-e2e > $O/bench_sp.json 2> $O/bench_sp.err; tail -3 $O/bench_sp.err
python -c "
import json; d=json.load(open('gpurun_out/bench_sp.json')); print(d['value'], d['time_to_T_s']); print(json.dumps(d['sparse_variant']))"
