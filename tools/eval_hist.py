"""Divergence histogram of k_eval (tuning build with -DKITC_EVAL_HIST): per (warp, far
cluster) how many of the batch's targets accept it, per (warp, leaf) how many sum it directly.
KITC_LIB=tools/variants/libkitc_hist.so python tools/eval_hist.py [config]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

cfg = KI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
X, W = KI.particles(cfg["N"], cfg["geometry"])
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
T = kitc.Tree(Xd, cfg["N0"])
fh = T.modified_weights(cfg["kernel"], cfg["n"], Wd)
T.eval(cfg["kernel"], cfg["n"], cfg["theta"], cfg["eps"], fh)
torch.cuda.synchronize()
h = (C.c_ulonglong * 10)()
kitc.lib().kitc_eval_hist(h)
far, near = list(h[:5]), list(h[5:])
print("far clusters per warp by #accepting targets (0..4):", far)
print("  lane-time share:", [round(k * 0 + far[k] / sum(far), 4) for k in range(5)],
      " idle-lane fraction of far work: %.4f" % (sum(far[k] * (4 - k) for k in range(5)) / (4 * sum(far))))
print("near leaves per warp by #participating targets (0..4):", near,
      " idle fraction: %.4f" % (sum(near[k] * (4 - k) for k in range(5)) / (4 * sum(near))))
