"""Per-source-line warp-stall samples of one kernel in an ncu report (ncu --page source --csv)."""
import csv, subprocess, sys, collections
rep, kid = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--print-kernel-base", "function", "-k", kid], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; agg = collections.Counter(); src = {}; hdr = None
reasons = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"): cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if not hdr or len(r) < 6: continue
    if not r[0]: continue
    try: samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError: continue
    key = (cur, r[0]); agg[key] += samp; src[key] = r[1].strip()[:70]
    for c in ("stall_barrier", "stall_short_sb", "stall_wait", "stall_long_sb", "stall_mio", "stall_math",
              "stall_branch_resolving", "stall_selected", "stall_not_selected", "stall_dispatch"):
        if c in hdr:
            try: reasons[key][c[6:]] += float(r[hdr.index(c)] or 0)
            except ValueError: pass
tot = sum(agg.values())
print("total samples", tot)
for key, v in agg.most_common(top):
    rs = " ".join("%s %d" % kv for kv in reasons[key].most_common(3) if kv[1] > 0)
    print("%6.0f %5.1f%%  %s:%s  %-70s [%s]" % (v, 100 * v / tot, key[0], key[1], src[key], rs))
