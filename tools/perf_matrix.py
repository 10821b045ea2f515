"""Eval throughput over (n, theta) on the C3 input (N = 1e6 uniform, N0 = 2000, Stokeslet and rotlet):
eval ms, pairs/target, % of the derived FP64 peak.  [PM_N=4,6 PM_THETA=0.7 PM_KERN=0] python tools/perf_matrix.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

FLOPS = {0: 32, 1: 59}
PEAK = 148 * 64 * 2 * 1965e6
X, W = KI.config_particles("C3")
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
G = kitc.Tree(Xd, 2000)
rows = []
NS = [int(v) for v in os.environ.get("PM_N", "4,6,8,10").split(",")]
THETAS = [float(v) for v in os.environ.get("PM_THETA", "0.5,0.7").split(",")]
for kern in [int(v) for v in os.environ.get("PM_KERN", "0,1").split(",")]:
    for n in NS:
        fh = G.modified_weights(kern, n, Wd)
        for theta in THETAS:
            out, st = G.eval(kern, n, theta, 0.01, fh, stats=True)
            pairs = int(st[:, 1].sum() + st[:, 3].sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            G.eval(kern, n, theta, 0.01, fh, out=out)
            e0.record()
            for _ in range(3):
                G.eval(kern, n, theta, 0.01, fh, out=out)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 3
            r = dict(kernel=kern, n=n, theta=theta, eval_ms=ms, pairs_per_target=pairs / 1e6,
                     frac=FLOPS[kern] * pairs / (ms * 1e-3) / PEAK)
            rows.append(r)
            print(json.dumps(r), flush=True)
