"""Time the O(N^2) direct kernel: python tools/bench_direct.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import kitc_inputs as KI  # noqa: E402
from paper_1902_02250_b200 import kitc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
X, W = KI.particles(N)
Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
out = kitc.direct(Xd, Wd, 0, 0.01)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    kitc.direct(Xd, Wd, 0, 0.01, out=out)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 3
pairs = N * (N - 1)
print(f"direct N={N}: {ms:.2f} ms, {pairs / ms / 1e6:.1f} Gpairs/s, {32 * pairs / ms / 1e9:.2f} TFLOP/s algorithmic "
      f"({32 * pairs / ms / 1e9 / 37.2249:.3f} of 37.22)")
