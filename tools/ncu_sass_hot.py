"""Per-region warp-stall samples from `ncu -i rep --page source --csv --print-source sass`.
Regions = loop bodies found from backward branches.  usage: python tools/ncu_sass_hot.py sass.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]])
    ins.append((a, r[ix["Source"]], int(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                int(r[ix["Instructions Executed"]] or 0), int(r[ix["Thread Instructions Executed"]] or 0),
                {k: float(r[i] or 0) for k, i in ix.items() if k.startswith("stall_") and "Not Issued" not in k}))
tot = sum(i[2] for i in ins)
loops = []
for a, src, *_ in ins:
    m = re.search(r"BRA\s+(?:`?\(?\.?L?_?x?_?)?(0x[0-9a-f]+)", src)
    if m:
        t = int(m.group(1), 16)
        if t < a:
            loops.append((t, a))
print(f"total samples {tot}")
for t, a in sorted(loops):
    sel = [i for i in ins if t <= i[0] <= a]
    s = sum(i[2] for i in sel)
    ex = sum(i[3] for i in sel)
    th = sum(i[4] for i in sel)
    st = {}
    for i in sel:
        for k, v in i[5].items():
            st[k] = st.get(k, 0) + v
    top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    fp = sum(i[3] for i in sel if re.match(r"\s*(@!?P\d\s+)?D(FMA|MUL|ADD)", i[1]))
    print(f"loop {t:#07x}-{a:#07x}: {100*s/tot:5.1f}% samples, {len(sel)} instr, warp-inst {ex:.3e}, "
          f"lanes/inst {th/max(ex,1):.1f}, fp64 warp-inst {fp:.3e}; " + ", ".join(f"{k[6:]} {100*v/max(s,1):.0f}%" for k, v in top))
