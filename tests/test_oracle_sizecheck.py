"""Oracle pins for the size-check variant (not in the
paper, motivated by its cost argument P:465-468): an accepted cluster with
N_C < (n+1)^3 particles is summed directly instead of through its proxies.

Pins:
  * (n+1)^3 > N: every accepted cluster is small -> the treecode is the direct
    sum (summation order only);
  * every cluster holds >= (n+1)^3 particles -> bitwise the plain treecode;
  * interaction lists brute-forced in Python at N <= 200 (coverage = N).
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O


def test_all_small_equals_direct():
    X, W = KI.particles(300, seed=3)
    T = O.Tree(X, 10)
    for K in (O.STOKESLET, O.ROTLET):
        u, st = T.treecode(K, 0.01, 6, 0.7, W, stats=True, size_check=True)   # 343 > 300
        assert st[:, 0].sum() == 0 and st[:, 2].sum() > 0
        assert O.rel_error(O.direct(K, 0.01, X, W), u) < 1e-13


def test_no_small_cluster_is_bitwise_plain():
    X, W = KI.particles(4000, seed=4)
    T = O.Tree(X, 100)
    assert (T.end - T.begin).min() >= 8
    F = T.modified_weights(W, 1)
    a = T.treecode(O.STOKESLET, 0.01, 1, 0.7, W, fhat=F)
    b = T.treecode(O.STOKESLET, 0.01, 1, 0.7, W, fhat=F, size_check=True)
    assert np.array_equal(a, b)


def _mac(lo, hi, x, tt):
    c = 0.5 * (lo + hi)
    h = 0.5 * (hi - lo)
    r2 = (h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]
    d = x - c
    R2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
    return R2 > 0.0 and r2 <= tt * R2


@pytest.mark.parametrize("N,N0,n", [(200, 8, 2), (180, 5, 1)])
def test_interaction_lists_brute_force_size_check(N, N0, n):
    X, W = KI.particles(N, seed=N0)
    T = O.Tree(X, N0)
    _, st = T.treecode(O.STOKESLET, 0.01, n, 0.7, W, stats=True, size_check=True)
    P3 = (n + 1) ** 3
    sz = T.end - T.begin
    anc = {0: []}
    for c in range(1, T.nclusters):
        anc[c] = anc[T.parent[c]] + [T.parent[c]]
    nsmall = 0
    for i in range(N):
        macs = [_mac(T.lo[c], T.hi[c], X[i], 0.7 * 0.7) for c in range(T.nclusters)]
        top = [c for c in range(T.nclusters) if macs[c] and not any(macs[a] for a in anc[c])]
        far = [c for c in top if sz[c] >= P3]
        small = [c for c in top if sz[c] < P3]
        near = [c for c in range(T.nclusters) if T.nchild[c] == 0 and not macs[c]
                and not any(macs[a] for a in anc[c])]
        direct = small + near
        covered = sum(sz[c] for c in far + direct)
        assert covered == N
        assert list(st[i]) == [len(far), len(far) * P3, len(direct), sum(sz[c] for c in direct) - 1, covered]
        nsmall += len(small)
    assert nsmall > 0


def test_targets_all_small_equals_direct():
    X, W = KI.particles(300, seed=3)
    Xt = np.random.default_rng(9).uniform(-2, 2, (80, 3))
    T = O.Tree(X, 10)
    u, st = T.treecode_targets(O.STOKESLET, 0.01, 6, 0.7, W, Xt, stats=True, size_check=True)
    assert st[:, 0].sum() == 0
    assert O.rel_error(O.direct_targets(O.STOKESLET, 0.01, X, W, Xt), u) < 1e-13
