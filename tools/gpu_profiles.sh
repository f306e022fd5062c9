#!/bin/bash
# gpurun: ncu captures for the round's profile summaries (one GPU, serial)
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
# 1) whole bench step set, launch list (cold, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant > /dev/null 2>&1
# 2) full sets: eigen kernels of one compression at k = 90, the congruence kernel and the
#    init square-tile int8 product (first launch), E pass (NVTX range)
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:"eig_|gram_congruence|oz_gemm|tall_small" -c 8 -o $O/step_final -f python tools/step_nvtx.py > $O/ncu_step.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_gemm_kernel -c 1 -o $O/oz_init -f python tools/init_only.py > $O/ncu_ozinit.log 2>&1
ls -la $O
