"""Concurrent kernel timeline of pipelined config-5 steps (CUPTI activity records through
torch.profiler: start/end of every kernel on both streams, no serialisation, warm caches).
Prints the critical-stream kernel sequence of the last steps with gaps, and per-kernel means."""
import json, os, sys, collections
sys.path.insert(0, '.')
import torch
import paper_1805_08990_b200 as dme
from workloads import make_config

prob = make_config(5)
s = dme.Solver(**dme.problem_kwargs(prob), h=0.005, rank_cap=64)
s.split_step("strang", "F12F3", 8)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.split_step("strang", "F12F3", 12)
    torch.cuda.synchronize()
path = "gpurun_out/kernel_trace.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
streams = collections.Counter(e["args"].get("stream") for e in ev)
print("streams", dict(streams))
def short(n):
    n = n.replace("void ", "").replace("(anonymous namespace)::", "").replace("dme::", "")
    return n.split("(")[0][:40]
# the step period: from consecutive gram_congruence launches
cong = [e for e in ev if "gram_congruence" in e["name"]]
per = [(b["ts"] - a["ts"]) for a, b in zip(cong, cong[1:])]
print("step periods (us):", " ".join("%.0f" % p for p in per), " mean %.1f" % (sum(per) / max(len(per), 1)))
# one full step in the middle: all kernels between two congruences
a, b = cong[len(cong) // 2], cong[len(cong) // 2 + 1]
print("\n%-40s %8s %8s %8s %6s" % ("kernel", "start", "dur", "end", "strm"))
for e in ev:
    if a["ts"] <= e["ts"] < b["ts"]:
        print("%-40s %8.1f %8.1f %8.1f %6s" % (short(e["name"]), e["ts"] - a["ts"], e["dur"], e["ts"] + e["dur"] - a["ts"], e["args"].get("stream")))
agg = collections.defaultdict(list)
for e in ev:
    agg[short(e["name"])].append(e["dur"])
print("\nper-kernel mean durations (us) over the traced steps")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print("%-40s n=%4d mean=%8.1f" % (k, len(v), sum(v) / len(v)))
