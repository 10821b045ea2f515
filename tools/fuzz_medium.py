"""GPU-vs-oracle fuzz at medium sizes (N 1e4..6e4): full GPU evaluation, oracle on 150 sampled
targets (its own full tree and modified weights), interaction counts and values at the gate.
python tools/fuzz_medium.py [cases]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
import oracle as O  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for case in range(cases):
    rng = np.random.default_rng(5000 + case + int(os.environ.get("FUZZ_OFFSET", "0")))
    kern = int(rng.integers(0, 3))
    geom = ["uniform", "sphere", "slab", "organisms"][int(rng.integers(0, 4))]
    if geom == "organisms":
        kern = 0
    N = int(rng.integers(5000, 30000)) * 2
    N0 = int(rng.choice([50, 200, 500, 1000, 2000]))
    n = int(rng.integers(1, 13))
    theta = float(rng.choice([0.5, 0.6, 0.7, 0.8]))
    eps = float(rng.choice([0.005, 0.01, 0.02]))
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=case, m=m)
    tg = KI.sample_targets(N, 150, seed=case)
    T = O.Tree(X, N0)
    F = T.modified_weights(W, n)
    ref, rst = T.treecode(kern, eps, n, theta, W, fhat=F, targets=tg, stats=True)
    G = kitc.Tree(torch.from_numpy(X).cuda(), N0)
    fh = G.modified_weights(kern, n, torch.from_numpy(W).cuda())
    got, gst = G.eval(kern, n, theta, eps, fh, stats=True)
    got, gst = got.cpu().numpy()[tg], gst.cpu().numpy()[tg]
    e = O.rel_error(ref, got)
    ok = np.array_equal(rst.astype(np.int64), gst) and e <= 1e-10
    bad += not ok
    print(f"{case:3d} kern {kern} {geom:9s} N {N:6d} N0 {N0:4d} n {n:2d} theta {theta} eps {eps}: "
          f"E_parity {e:.2e} counts {'ok' if np.array_equal(rst.astype(np.int64), gst) else 'DIFF'}", flush=True)
print(f"failures {bad} of {cases}")
