for v in default; do
  if [ $v = default ]; then unset KITC_LIB; else export KITC_LIB=$PWD/tools/variants/libkitc_$v.so; fi
  python - <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
import kitc_inputs as KI
from paper_1902_02250_b200 import kitc
X, W = KI.config_particles("C2")
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
G = kitc.Tree(Xd, 500)
res = []
for n in (1, 2, 3, 4, 5, 6, 9, 10):
    fh = G.modified_weights(0, n, Wd)
    out = G.eval(0, n, 0.7, 0.01, fh)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(6):
        e0.record(); G.eval(0, n, 0.7, 0.01, fh, out=out); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    res.append("n=%d %.3f ms" % (n, sorted(ts)[3]))
print(os.environ.get("KITC_LIB", "default")[-20:], " ".join(res))
PY
done
