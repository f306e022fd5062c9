#!/bin/bash
# gpurun: round-2 ncu evidence: launch list of the bench (cold, serialised), full sets of the step
# kernels (E pass, eigen passes, complement basis, tail kernels), the E pass alone (dram bytes)
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-variant --no-sparse --no-pade > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "step/" -k regex:"eig_|gram_congruence|oz_gemm|tall_small|complement|tail_assemble|gemm_nt|splitk" -c 16 -o $O/r02_step -f python tools/step_nvtx.py > $O/ncu_step.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "epass/" -k regex:oz_gemm -c 1 -o $O/r02_epass -f python tools/epass_one.py 53 > $O/ncu_epass.log 2>&1
ls -la $O/*.ncu-rep
