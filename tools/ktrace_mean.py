"""Per-kernel mean durations and the step period from a chrome trace written by kernel_trace_cfg.py."""
import json, sys, collections
ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"] if e.get("cat") == "kernel"]
agg = collections.defaultdict(list)
for e in ev:
    n = e["name"].replace("void ", "").replace("(anonymous namespace)::", "").replace("dme::", "").split("(")[0][:44]
    agg[n].append(e["dur"])
span = max(e["ts"] + e["dur"] for e in ev) - min(e["ts"] for e in ev)
print("span %.1f us" % span)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print("%-44s n=%3d mean=%7.1f sum=%8.1f" % (k, len(v), sum(v) / len(v), sum(v)))
