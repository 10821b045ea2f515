"""One C3 step (tree + weights + eval) for ncu captures: python tools/profile_step.py [config] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

cfg = KI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X, W = KI.particles(cfg["N"], cfg["geometry"])
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
T = kitc.Tree(Xd, cfg["N0"])
out = torch.zeros((cfg["N"], kitc.kitc_kernel_dims(cfg["kernel"])[1]), dtype=torch.float64, device="cuda")
for _ in range(reps):
    T.build(Xd, cfg["N0"])
    fh = T.modified_weights(cfg["kernel"], cfg["n"], Wd, cluster_range=(1, T.nclusters))
    T.eval(cfg["kernel"], cfg["n"], cfg["theta"], cfg["eps"], fh, out=out)
torch.cuda.synchronize()
print("ok", out.abs().sum().item())
