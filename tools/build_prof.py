"""Phase times inside the cooperative tree build (tuning build with -DKITC_BUILD_PROF):
KITC_LIB=tools/variants/libkitc_bprof.so python tools/build_prof.py [config]"""
import collections
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

cfg = KI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
X, _ = KI.particles(cfg["N"], cfg["geometry"])
Xd = torch.from_numpy(X).cuda()
T = kitc.Tree(Xd, cfg["N0"])
L = kitc.lib()
buf = (C.c_ulonglong * 1024)()
L.kitc_build_prof(buf, 1024)   # drop the first build's records
for _ in range(3):
    T.build(Xd, cfg["N0"])
n = L.kitc_build_prof(buf, 1024)
recs = [(v >> 56, v & ((1 << 56) - 1)) for v in buf[:n]]
# one build = records from tag 0 to the last tag 23; take the last build
starts = [i for i, (t, _) in enumerate(recs) if t == 0]
last = recs[starts[-1]:]
names = {0: "stage+root box", 10: "SB box partials", 11: "S1 box/split", 12: "S2 scan", 13: "S3 counts",
         14: "S4 offsets", 15: "S5 children", 16: "S6 scatter", 20: "S7+tail", 21: "bottom-up", 22: "init",
         23: "top-down", 30: "leaf Morton order"}
agg = collections.OrderedDict()
for (t0, a), (t1, b) in zip(last, last[1:]):
    agg.setdefault(names.get(t1, str(t1)), [0, 0])
    agg[names.get(t1, str(t1))][0] += 1
    agg[names.get(t1, str(t1))][1] += (b - a) / 1e3
tot = (last[-1][1] - last[0][1]) / 1e3
print(f"build phases (us), {cfg['N']} particles, barriers {len(last)}: total {tot:.1f} us between first and last barrier")
for k, (c, us) in agg.items():
    print(f"  {k:18s} x{c:3d} {us:9.1f} us")
