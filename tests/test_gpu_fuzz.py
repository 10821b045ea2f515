"""Seeded random configurations (sizes, leaf sizes, degrees, MAC parameters, kernels,
geometries, eps, self term, separate targets, the size-check variant): GPU treecode vs the
oracle at the parity gate, interaction counts equal.  Small cases, many code paths (ragged
leaves and batches, partial fhat blocks, runtime-P kernel, lane teams)."""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TREE_GATE = 1e-10


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1902_02250_b200 import kitc
    return kitc


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("case", range(14))
def test_fuzz(K, case):
    rng = np.random.default_rng(1000 + case)
    kern = int(rng.integers(0, 3))
    geom = ["uniform", "sphere", "slab"][int(rng.integers(0, 3))]
    N = int(rng.integers(1, 2500))
    N0 = int(rng.integers(1, 150))
    n = int(rng.integers(1, 11))
    theta = float(rng.choice([0.0, 0.3, 0.5, 0.7, 0.9]))
    eps = float(rng.choice([0.005, 0.02, 0.1]))
    self_omit = bool(rng.integers(0, 2))
    size_check = bool(rng.integers(0, 2))
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=case, m=m)
    T = O.Tree(X, N0)
    F = T.modified_weights(W, n)
    ref, rst = T.treecode(kern, eps, n, theta, W, fhat=F, self_omit=self_omit, stats=True, size_check=size_check)
    G = K.Tree(dev(X), N0)
    fh = G.modified_weights(kern, n, dev(W))
    got, gst = G.eval(kern, n, theta, eps, fh, self_omit=self_omit, stats=True, size_check=size_check)
    torch.cuda.synchronize()
    got, gst = got.cpu().numpy(), gst.cpu().numpy()
    assert np.array_equal(rst.astype(np.int64), gst)
    if np.any(ref != 0):
        assert O.rel_error(ref, got) <= TREE_GATE, (kern, geom, N, N0, n, theta, eps, self_omit, size_check)
    # separate targets, same tree
    Xt = rng.uniform(-1.6, 1.6, (int(rng.integers(1, 700)), 3))
    reft, rstt = T.treecode_targets(kern, eps, n, theta, W, Xt, fhat=F, stats=True, size_check=size_check)
    gott, gstt = G.eval_targets(kern, n, theta, eps, fh, dev(Xt), stats=True, size_check=size_check)
    torch.cuda.synchronize()
    assert np.array_equal(rstt.astype(np.int64), gstt.cpu().numpy())
    assert O.rel_error(reft, gott.cpu().numpy()) <= TREE_GATE
