import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import kitc_inputs as KI, oracle as O
from paper_1902_02250_b200 import kitc
for name in ("X1", "X1L"):
    c = KI.CONFIGS[name]
    X, W = KI.config_particles(name)
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    u = kitc.treecode(Xd, Wd, 0, c["n"], c["theta"], c["N0"], c["eps"]).cpu().numpy()
    tg = KI.sample_targets(c["N"], 200, seed=3)
    t0 = time.time()
    d_or = O.direct(0, c["eps"], X, W, targets=tg)
    d_gpu = kitc.direct_sample(Xd, Wd, 0, c["eps"], torch.from_numpy(tg).cuda()).cpu().numpy()
    print(name, "oracle direct sample %.1fs" % (time.time() - t0), "GPU direct vs oracle %.2e" % O.rel_error(d_or, d_gpu),
          "E_sample(treecode vs oracle direct) %.3e" % O.rel_error(d_or, u[tg]))
    # per-target relative errors: what dominates?
    e = np.linalg.norm(u[tg] - d_or, axis=1) / np.linalg.norm(d_or, axis=1)
    print("   per-target rel err: median %.2e  90%% %.2e  max %.2e; |u_d| median %.3f max %.3f" % (
        np.median(e), np.percentile(e, 90), e.max(), np.median(np.linalg.norm(d_or, axis=1)), np.linalg.norm(d_or, axis=1).max()))
