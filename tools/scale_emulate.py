"""Per-rank work of the k-GPU decomposition, timed on ONE GPU (no collective, no peers):
for k in 1, 2, 4, 8, each rank's share -- its cluster shard of the modified weights and its
interleaved part of the evaluation (kitc_eval_part) -- runs alone on the device and is timed with
CUDA events; the projected k-GPU step = replicated build + max over ranks (weights shard) + max over
ranks (eval part).  Exchange and barrier costs are NOT included (this node has one GPU); the point is
the Amdahl terms and the load balance of the decomposition.
python tools/scale_emulate.py [config] [reps]"""
import json
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
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = KI.CONFIGS[name]
X, W = KI.config_particles(name)
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
T = kitc.Tree(Xd, c["N0"])
kern, n = c["kernel"], c["n"]
p = kitc.kitc_kernel_dims(kern)[1]
fh = torch.zeros(T.fhat_shape(kern, n), dtype=torch.float64, device="cuda")
out = torch.zeros((c["N"], p), dtype=torch.float64, device="cuda")
rg = T.export_ranges()


def timed(fn):
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


t_build = timed(lambda: T.build(Xd, c["N0"]))
T.modified_weights(kern, n, Wd, cluster_range=(1, T.nclusters), fhat=fh)
res = {"config": name, "build_ms": t_build, "ranks": {}}
base = None
for k in (1, 2, 4, 8):
    shards = D.cluster_shards(rg["begin"], rg["end"], k, skip_root=True)
    tw = [timed(lambda cb=cb, ce=ce: T.modified_weights(kern, n, Wd, cluster_range=(cb, ce), fhat=fh))
          for cb, ce in shards]
    te = [timed(lambda r=r: T.eval(kern, n, c["theta"], c["eps"], fh, out=out, part=(r, k))) for r in range(k)]
    step = t_build + max(tw) + max(te)
    if base is None:
        base = step
    res["ranks"][k] = {"weights_ms_max": max(tw), "eval_ms_max": max(te), "eval_ms_mean": float(np.mean(te)),
                       "eval_imbalance": max(te) / float(np.mean(te)) - 1.0, "projected_step_ms": step,
                       "projected_targets_per_s": c["N"] / (step * 1e-3),
                       "projected_efficiency": base / (k * step)}
    print(json.dumps({"k": k, **res["ranks"][k]}), flush=True)
print(json.dumps(res))
