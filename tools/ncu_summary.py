"""Summarise ncu outputs for profiles/: python tools/ncu_summary.py rep.ncu-rep|launches.csv [...]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__sass_inst_executed_op_shared_ld.sum"]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, zip(vals, units)))
        print(f"== kernel: {d.get('Kernel Name', ('?',))[0]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][0]} {d[k][1]}")
        st = sorted(((float(v[0]), k) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")),
                    reverse=True)[:8]
        print("  top stall reasons (warps per issue):")
        for v, k in st:
            print(f"    {v:6.3f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        k = r[iK].split("(")[0].replace("void ", "").replace("kitc::<unnamed>::", "")
        v = float(r[iV].replace(",", ""))
        v = v / 1e3 if r[iU] == "ns" else v * 1e3 if r[iU] == "ms" else v
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for k, (n, t) in agg.items():
        print(f"{k[:44]:44s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}%")


for p in sys.argv[1:]:
    print(f"# {p}")
    (rep if p.endswith(".ncu-rep") else launches)(p)
