"""Per-source-line warp-stall samples of an ncu report (needs -lineinfo + --import-source):
python tools/ncu_lines.py REP.ncu-rep [top]  -> top lines and totals per function region."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr = None, None
agg = collections.OrderedDict()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[-(len(hdr) - 2):]))   # source text may hold unescaped quotes: align from the right
    key = (cur, int(r[0]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        ex = int(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        continue
    a = agg.setdefault(key, [0, 0, r[1][:90]])
    a[0] += s
    a[1] += ex
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}")
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% {ex:12.3e}  {f}:{ln:<4d} {src}")
# regions: function bodies by line range (eval.cu), from the source text
regions = collections.Counter()
src = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
if src:
    starts = [(i + 1, m.group(1)) for i, l in enumerate(src) for m in [re.search(r"^\S.*\b(\w+)\(", l)] if m and "__device__" in (src[i - 1] if i else "") + l or (m and "__global__" in l)]
    starts.sort()
    for (f, ln), (s, ex, _) in agg.items():
        if f != src and f == "eval.cu":
            name = "?"
            for st, nm in starts:
                if st <= ln:
                    name = nm
            regions[name] += s
        else:
            regions[f] += s
    for k, v in regions.most_common():
        print(f"{100 * v / tot:5.1f}%  {k}")
