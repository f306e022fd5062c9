#!/bin/bash
# One gpurun call refreshing the round's evidence: build, GPU tests, smoke, bench (config 5 and 6),
# reference arm, ncu launch list of a short bench run, full captures of the step kernels.
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench5.json 2> $O/bench5.err
timeout 600 python bench.py --config 6 > $O/bench6.json 2> $O/bench6.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:"eig_|gram_congruence|oz_gemm|tall_small" -c 8 -o $O/step_final -f python tools/step_nvtx.py > $O/ncu_step.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/bench5.json $O/bench6.json $O/bench_ref.json
