#!/bin/bash
# One gpurun call: build check, GPU tests, smoke, bench, ncu launch list + one full capture of the
# E-pass kernel. Everything lands in gpurun_out/.
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "epass/" -k regex:oz_gemm -c 1 -o $O/epass_oz -f python tools/epass_one.py 56 > $O/ncu_full.log 2>&1
