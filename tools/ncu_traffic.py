"""Record one k_eval launch's DRAM traffic from an `ncu --set full` report into
profiles/ncu_traffic.json (the bench's roofline.traffic), tagged with the build id
of the library that was captured:  python tools/ncu_traffic.py CONFIG REP.ncu-rep BUILD_ID SUMMARY_PATH"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, rep, bid, summ = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
d = dict(zip(hdr, zip(rows[2], units)))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * scale[d["dram__bytes_read.sum"][1]]
wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * scale[d["dram__bytes_write.sum"][1]]
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
tab = json.load(open(path)) if os.path.exists(path) else {}
tab[cfg] = {"kernel": d["Kernel Name"][0].split("(")[0], "dram_bytes_per_launch": int(rd + wr), "build_id": bid,
            "source": f"{summ} (dram__bytes_read.sum {rd / 1e6:.3f} MB + dram__bytes_write.sum {wr / 1e6:.3f} MB)"}
json.dump(tab, open(path, "w"), indent=1)
print(json.dumps(tab[cfg]))
