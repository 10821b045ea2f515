"""Small end-to-end exercise of every entry point, for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
for (N, N0, n, kern, geom) in [(3001, 60, 8, 0, "uniform"), (2000, 40, 4, 1, "sphere"), (3775, 100, 7, 2, "rods"),
                               (1500, 30, 12, 0, "uniform"), (7, 1, 2, 0, "uniform")]:
    m = 6 if kern == 2 else 3
    X, W = KI.particles(N, geom, seed=1, m=m)
    G = kitc.Tree(dev(X), N0)
    fh = G.modified_weights(kern, n, dev(W))
    u, st = G.eval(kern, n, 0.7, 0.02, fh, stats=True)
    G.eval(kern, n, 0.7, 0.02, fh, size_check=True)
    G.eval(kern, n, 0.7, 0.02, fh, part=(1, 3))
    Xt = np.random.default_rng(2).uniform(-1.5, 1.5, (513, 3))
    G.eval_targets(kern, n, 0.7, 0.02, fh, dev(Xt), stats=True)
    reps = [torch.zeros_like(fh) for _ in range(2)]
    kitc.kitc_modified_weights_peers(G.handle, kern, n, kitc._ptr(dev(W)), 0, G.nclusters,
                                     [r.data_ptr() for r in reps], kitc._stream())
    d = kitc.direct(dev(X), dev(W), kern, 0.02)
    kitc.direct_sample(dev(X), dev(W), kern, 0.02, torch.arange(0, N, 3, device="cuda"))
    print(N, geom, "E", kitc.rel_error(d, u))
torch.cuda.synchronize()
print("sanitize run ok, build flags", kitc.kitc_build_flags(), "library", kitc.LIB_PATH)
