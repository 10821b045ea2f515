"""Warp-stall samples and FP64 instructions of the k_eval capture by code region (eval.cu / pair.cuh
line ranges): python tools/ncu_regions.py REP.ncu-rep"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
NAMES = {"tma_round": "TMA / mbarrier helpers", "mbar_wait": "TMA / mbarrier helpers",
         "smem_u32": "TMA / mbarrier helpers", "far_field": "far field: staging, row setup, stage loop",
         "far_field_team": "far field teams (1-2 accepting targets)",
         "near_field_tb": "near field loop, target pairs (loads)", "near_field_impl": "near field loop (loads)",
         "near_field": "near field dispatch / teams", "near_leaf": "near field dispatch / teams",
         "k_eval": "traversal (MAC, stack, epilogue)", "__launch_bounds__": "traversal (MAC, stack, epilogue)"}
# function of every line of eval.cu (the source the capture was built from): the last definition above it
EVAL = []
for i, ln in enumerate(open(__import__("os").path.join(ROOT, "paper_1902_02250_b200", "csrc", "eval.cu")), 1):
    m = re.search(r"__(?:device|global)__.*?\b(\w+)\(", ln)
    if m and not ln.lstrip().startswith("//"):
        EVAL.append((i, m.group(1)))


def region(f, ln):
    if f == "pair.cuh":
        if 40 <= ln <= 44:
            return "s^-1/2 (MUFU seed + Newton)"
        if 182 <= ln <= 194:
            return "pair math, near field / partial rows"
        if 198 <= ln <= 214:
            return "pair math, far field rows"
        return "pair.cuh other"
    if f == "eval.cu":
        name = None
        for start, fn in EVAL:
            if start <= ln:
                name = fn
        return NAMES.get(name, "eval.cu: " + str(name))
    return "other (" + f + ")"


samp, fp, stalls = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
cur = hdr = reg = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr[2:], r[-(len(hdr) - 2):]))
    if r[0].isdigit():
        reg = region(cur, int(r[0]))
        try:
            samp[reg] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            pass
        continue
    try:
        ex = int(d.get("Instructions Executed") or 0)
    except ValueError:
        continue
    ops = [o for o in (r[3].split() if len(r) > 3 else []) if not o.startswith("@")]
    if ops and re.match(r"D(FMA|MUL|ADD)", ops[0]):
        fp[reg] += ex
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[reg][k[6:]] += float(v or 0)
            except ValueError:
                pass
ts, tf = sum(samp.values()), sum(fp.values())
print(f"# {sys.argv[1]}: warp-stall samples {ts}, FP64 warp instructions {tf}")
print(f"{'region':44s} {'samples':>8s} {'FP64 inst':>9s}  top stalls")
for k, v in samp.most_common():
    st = stalls[k]
    tot = sum(st.values()) or 1
    top = ", ".join(f"{n} {100 * x / tot:.0f}%" for n, x in st.most_common(3))
    print(f"{k:44s} {100 * v / ts:7.1f}% {100 * fp[k] / max(tf, 1):8.1f}%  {top}")
