"""kitc_eval_targets throughput on the C3 tree: 1e6 separate uniform targets in [-1,1]^3 vs the
targets = sources evaluation.  python tools/bench_targets.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

c = KI.CONFIGS["C3"]
X, W = KI.config_particles("C3")
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
Xt = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, (c["N"], 3))).cuda()
G = kitc.Tree(Xd, c["N0"])
fh = G.modified_weights(0, c["n"], Wd)
out = G.eval(0, c["n"], c["theta"], c["eps"], fh)
outt = G.eval_targets(0, c["n"], c["theta"], c["eps"], fh, Xt)
_, st = G.eval_targets(0, c["n"], c["theta"], c["eps"], fh, Xt, stats=True)
pairs = int(st[:, 1].sum() + st[:, 3].sum())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("sources as targets", lambda: G.eval(0, c["n"], c["theta"], c["eps"], fh, out=out)),
                 ("1e6 separate targets", lambda: G.eval_targets(0, c["n"], c["theta"], c["eps"], fh, Xt, out=outt))):
    fn()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.2f} ms, {c['N'] / ms / 1e3:.3g} Mtargets/s")
print(f"separate targets: {pairs / c['N']:.0f} pairs/target, {32 * pairs / 37.22e12 * 1e3:.1f} ms at 100% of the FP64 peak")
