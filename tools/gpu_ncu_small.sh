#!/bin/bash
# gpurun: ncu full sets with dense PC sampling of the one-CTA step kernels in the pipelined config-5 run
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none \
  -k regex:"eig_tri|eig_vec|eig_fin|complement_basis|tail_assemble|gram_congruence|proj_gram" \
  --launch-skip 40 --launch-count 10 -o $O/small_kernels -f python tools/pipe_probe.py > $O/ncu_small.log 2>&1
tail -3 $O/ncu_small.log
