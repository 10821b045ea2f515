"""Per-rank work balance of the multi-GPU target split (uses the library's exact per-target
interaction counts): contiguous batch ranges balanced by target count vs chunk-interleaved.
python tools/balance_check.py [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import dist as D  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = KI.CONFIGS[name]
X, W = KI.config_particles(name)
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
T = kitc.Tree(Xd, cfg["N0"])
fh = T.modified_weights(cfg["kernel"], cfg["n"], Wd)
_, st = T.eval(cfg["kernel"], cfg["n"], cfg["theta"], cfg["eps"], fh, stats=True)
st = st.cpu().numpy()
perm = T.export()["perm"]
cost_t = 16.0 * st[:, 1] + 22.0 * st[:, 3]           # FP64 instructions per target (far, near pairs)
cost_sorted = cost_t[perm]                            # by sorted position
nb = T.nbatches
prefix = np.array([T.batch_targets(b) for b in range(nb + 1)])
bcost = np.add.reduceat(cost_sorted, prefix[:-1]) if nb else np.zeros(0)
for k in (2, 4, 8):
    sh = D.batch_shards(prefix, k)
    w = [bcost[b:e].sum() for b, e in sh]
    CH = 64
    wi = np.zeros(k)
    for c0 in range(0, nb, CH):
        wi[(c0 // CH) % k] += bcost[c0:c0 + CH].sum()
    print(f"{name} k={k}: contiguous max/mean {max(w) / np.mean(w):.4f}   interleaved(64) max/mean {wi.max() / wi.mean():.4f}")
