"""Per-phase device (CUDA events) and host (wall) times of one step: build, weights, eval.
python tools/phase_times.py [config] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

cfg = KI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
X, W = KI.particles(cfg["N"], cfg["geometry"], m=6 if cfg["kernel"] == 2 else 3)
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
T = kitc.Tree(Xd, cfg["N0"])
p = kitc.kitc_kernel_dims(cfg["kernel"])[1]
out = torch.zeros((cfg["N"], p), dtype=torch.float64, device="cuda")
fh = torch.zeros(T.fhat_shape(cfg["kernel"], cfg["n"]), dtype=torch.float64, device="cuda")
rows = []
for r in range(reps + 2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    ev[0].record()
    T.build(Xd, cfg["N0"])
    h1 = time.perf_counter()
    ev[1].record()
    T.modified_weights(cfg["kernel"], cfg["n"], Wd, cluster_range=(1, T.nclusters), fhat=fh)
    h2 = time.perf_counter()
    ev[2].record()
    T.eval(cfg["kernel"], cfg["n"], cfg["theta"], cfg["eps"], fh, out=out)
    h3 = time.perf_counter()
    ev[3].record()
    ev[3].synchronize()
    h4 = time.perf_counter()
    if r >= 2:
        rows.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                     ev[0].elapsed_time(ev[3]), 1e3 * (h1 - h0), 1e3 * (h2 - h1), 1e3 * (h3 - h2), 1e3 * (h4 - h0)])
m = np.median(np.array(rows), axis=0)
print("median ms: dev build %.3f weights %.3f eval %.3f total %.3f | host build %.3f weights %.3f eval-enqueue %.3f total %.3f"
      % tuple(m))
