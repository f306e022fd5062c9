"""Per-kernel time of the last timed steps in an ncu launch list (gpu__time_duration.sum)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
data = [(r[ki].split('(')[0][-48:], float(r[vi].replace(',', ''))) for r in rows[1:]]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in data[-last:]:
    print(f"  {k:48s} {v/1e3:8.1f} us")
