"""BASELINE config C2: N = 1e5 uniform Stokeslet, N0 = 500, eps = 0.01; sweep n = 1..10 at
theta in {0.5, 0.7}: relative 2-norm error E vs the direct sum and GPU time per n, with the
oracle's E on a target sample beside the GPU's E on the same sample (the north star's
"GPU error tracks the oracle's error-vs-n curve").  Writes one JSON document to stdout.

  python tools/sweep_c2.py [--sample 300] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
import oracle as O  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sample", type=int, default=300)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

c = KI.CONFIGS["C2"]
N, N0, eps = c["N"], c["N0"], c["eps"]
X, W = KI.config_particles("C2")
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
ref = kitc.direct(Xd, Wd, 0, eps)
tg = KI.sample_targets(N, args.sample, seed=5)
d_or = O.direct(0, eps, X, W, targets=tg)
T_or = O.Tree(X, N0)
G = kitc.Tree(Xd, N0)
out = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
rows = []
for theta in (0.5, 0.7):
    for n in range(1, 11):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ts, te = [], []
        for r in range(args.reps + 1):
            ev[0].record()
            G.build(Xd, N0)
            fh = G.modified_weights(0, n, Wd, cluster_range=(1, G.nclusters))
            ev[1].record()
            G.eval(0, n, theta, eps, fh, out=out)
            ev[2].record()
            ev[2].synchronize()
            if r:
                ts.append(ev[0].elapsed_time(ev[2]))
                te.append(ev[1].elapsed_time(ev[2]))
        E_gpu = kitc.rel_error(ref, out)
        got = out.cpu().numpy()
        F_or = T_or.modified_weights(W, n)
        u_or, st = T_or.treecode(0, eps, n, theta, W, fhat=F_or, targets=tg, stats=True)
        row = dict(theta=theta, n=n, E_gpu_all=E_gpu,
                   E_gpu_sample=O.rel_error(d_or, got[tg]), E_oracle_sample=O.rel_error(d_or, u_or),
                   gpu_vs_oracle_sample=O.rel_error(u_or, got[tg]),
                   step_ms_median=float(np.median(ts)), eval_ms_median=float(np.median(te)),
                   pairs_per_target_sample=float((st[:, 1] + st[:, 3]).mean()))
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
kitc.direct(Xd, Wd, 0, eps, out=out)
t1.record()
t1.synchronize()
print(json.dumps({"config": "C2", "N": N, "N0": N0, "eps": eps, "sample_targets": int(len(tg)),
                  "direct_ms": t0.elapsed_time(t1), "rows": rows}, indent=1))
