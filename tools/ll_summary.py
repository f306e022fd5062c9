"""Per-kernel median durations over the last N launches of an ncu launch list (csv)."""
import csv, sys, statistics
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
tail = rows[-int(sys.argv[2]) if len(sys.argv) > 2 else 0:]
g = defaultdict(list)
for r in tail:
    g[r[4].split('(')[0][-48:] + ' ' + r[8]].append(float(r[-1]) / 1000)
for k, v in sorted(g.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:62s} n={len(v):4d} med={statistics.median(v):8.1f} us")
