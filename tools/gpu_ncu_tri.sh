#!/bin/bash
O=gpurun_out; mkdir -p $O
for g in 7 16; do
  timeout 300 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "probe/" -k regex:"eig_(tri|vec)_kernel" -o $O/tri_g$g -f python tools/tri_one.py $g > $O/ncu_tri_g$g.log 2>&1
  tail -3 $O/ncu_tri_g$g.log
done
ls -la $O
