"""Concurrent kernel timeline of a few steps of config argv[1] (CUPTI via torch.profiler): the
kernel sequence of the last traced step(s) with start offsets and gaps."""
import json, os, sys, collections
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config
cfg = int(sys.argv[1])
R = {1: ("lie", "F1F2", 0.001), 2: ("strang", "F12", 0.005), 3: ("strang", "F12F3", 0.005),
     4: ("strang", "F12F3F4", 0.005), 5: ("strang", "F12F3", 0.005)}[cfg]
prob = make_config(cfg)
s = dme.Solver(**dme.problem_kwargs(prob), h=R[2], rank_cap=64)
s.split_step(R[0], R[1], 5)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.split_step(R[0], R[1], 3)
    torch.cuda.synchronize()
path = "gpurun_out/kernel_trace_c%d.json" % cfg
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
def short(n):
    n = n.replace("void ", "").replace("(anonymous namespace)::", "").replace("dme::", "")
    return n.split("(")[0][:40]
t0 = ev[0]["ts"]
prev_end = t0
print("%-40s %8s %7s %6s %5s" % ("kernel", "start", "dur", "gap", "strm"))
for e in ev:
    print("%-40s %8.1f %7.1f %6.1f %5s" % (short(e["name"]), e["ts"] - t0, e["dur"], e["ts"] - prev_end, e["args"].get("stream")))
    prev_end = max(prev_end, e["ts"] + e["dur"])
print("total %.1f us for 3 steps" % (prev_end - t0))
