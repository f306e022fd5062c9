O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --no-cpu --no-variant > $O/bench_sp.json 2> $O/bench_sp.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cheb_reg_kernel -c 1 -o $O/cheb_one -f python tools/cheb_one.py 46 > $O/ncu_cheb.log 2>&1
ncu -i $O/cheb_one.ncu-rep --page details > $O/cheb_details.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_sp.json')); print(d['value'], d['time_to_T_s']); print(json.dumps(d['sparse_variant']))"
