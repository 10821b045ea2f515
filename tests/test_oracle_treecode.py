"""Oracle pins: treecode traversal, far field, direct sum and E
(Algorithm 2, Eq. pc_approximation_3D, Eq. N-body P:42-67,
Eq. error).

Pins:
  * theta = 0 -> treecode == direct sum (only zero-radius clusters accepted,
    exact by reading A14);
  * a polynomial test kernel of degree <= n per source coordinate makes the far
    field exact -> treecode == direct at theta = 0.7;
  * coverage and interaction lists brute-forced in Python at N <= 200
    (MAC evaluated in Python floats, RN, no FMA -> identical decisions);
  * E(n) decreases geometrically (Chebyshev rate bound);
  * direct sum vs an independent numpy evaluation, self-term closed form,
    permutation invariance; E closed forms.
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O


def test_theta_zero_equals_direct():
    for K in [O.STOKESLET, O.ROTLET]:
        X, W = KI.particles(400, seed=5)
        T = O.Tree(X, 10)
        for n in [1, 3]:
            u = T.treecode(K, 0.01, n, 0.0, W)
            d = O.direct(K, 0.01, X, W)
            assert O.rel_error(d, u) < 1e-13


def test_polynomial_kernel_far_field_exact():
    X, _ = KI.particles(1500, seed=6)
    W = np.random.default_rng(6).uniform(-1, 1, (1500, 1))
    T = O.Tree(X, 40)
    for n in [2, 3, 4]:
        u, st = T.treecode(O.POLY, 0.0, n, 0.7, W, stats=True)
        assert st[:, 0].sum() > 0                              # far field really used
        d = O.direct(O.POLY, 0.0, X, W, poly_deg=n)
        assert O.rel_error(d, u) < 1e-12


def _mac(lo, hi, x, tt):
    c = 0.5 * (lo + hi)
    h = 0.5 * (hi - lo)
    r2 = (h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]
    d = x - c
    R2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
    return R2 > 0.0 and r2 <= tt * R2


@pytest.mark.parametrize("N,N0,theta", [(200, 8, 0.7), (150, 3, 0.5), (200, 20, 0.9)])
def test_interaction_lists_brute_force(N, N0, theta):
    X, W = KI.particles(N, seed=N0)
    T = O.Tree(X, N0)
    n = 3
    _, st = T.treecode(O.STOKESLET, 0.01, n, theta, W, stats=True)
    Xs = X[T.perm]
    iperm = np.argsort(T.perm)
    tt = theta * theta
    anc = {0: []}
    for c in range(1, T.nclusters):
        anc[c] = anc[T.parent[c]] + [T.parent[c]]
    for i in range(N):
        x = X[i]
        macs = [_mac(T.lo[c], T.hi[c], x, tt) for c in range(T.nclusters)]
        far = [c for c in range(T.nclusters) if macs[c] and not any(macs[a] for a in anc[c])]
        near = [c for c in range(T.nclusters) if T.nchild[c] == 0 and not macs[c]
                and not any(macs[a] for a in anc[c])]
        nfar_pairs = len(far) * (n + 1) ** 3
        covered = sum(T.end[c] - T.begin[c] for c in far + near)
        near_pairs = sum(T.end[c] - T.begin[c] for c in near) - 1   # self omitted
        assert covered == N                                   # every source exactly once
        assert list(st[i]) == [len(far), nfar_pairs, len(near), near_pairs, covered]
        own_leaf = [c for c in near if T.begin[c] <= iperm[i] < T.end[c]]
        assert len(own_leaf) == 1                             # own cluster never accepted


def test_error_decreases_geometrically_with_n():
    X, W = KI.particles(1000, seed=0)
    T = O.Tree(X, 100)
    d = O.direct(O.STOKESLET, 0.01, X, W)
    E = [O.rel_error(d, T.treecode(O.STOKESLET, 0.01, n, 0.7, W)) for n in range(1, 11)]
    assert all(E[i + 1] < E[i] for i in range(len(E) - 1))
    # Bernstein-ellipse bound for theta = 0.7: >= 0.389 decades per degree
    slope = (np.log10(E[1]) - np.log10(E[9])) / 8
    assert slope > 0.389
    # theta = 0.5 converges faster than 0.7 at the same n
    E5 = O.rel_error(d, T.treecode(O.STOKESLET, 0.01, 6, 0.5, W))
    assert E5 < E[5]


def test_rotlet_error_decreases():
    X, W = KI.particles(800, seed=1)
    T = O.Tree(X, 60)
    d = O.direct(O.ROTLET, 0.01, X, W)
    E = [O.rel_error(d, T.treecode(O.ROTLET, 0.01, n, 0.7, W)) for n in (2, 4, 6, 8)]
    assert all(E[i + 1] < E[i] for i in range(3))


def test_single_leaf_equals_direct_and_self_term():
    X, W = KI.particles(300, seed=8)
    T = O.Tree(X, 300)
    assert T.nclusters == 1
    for K in [O.STOKESLET, O.ROTLET]:
        assert O.rel_error(O.direct(K, 0.02, X, W), T.treecode(K, 0.02, 4, 0.7, W)) < 1e-14
    inc = O.direct(O.STOKESLET, 0.02, X, W, self_omit=False)
    omt = O.direct(O.STOKESLET, 0.02, X, W, self_omit=True)
    H1_0 = 1.0 / (4 * np.pi * 0.02)                           # Eq. MRS_kernels at r = 0
    assert np.allclose(inc - omt, W * H1_0, rtol=1e-10, atol=1e-12)
    tinc = T.treecode(O.STOKESLET, 0.02, 4, 0.7, W, self_omit=False)
    assert np.allclose(tinc, inc, rtol=1e-12, atol=1e-12)


def _numpy_stokeslet(X, W, eps):
    d = X[:, None, :] - X[None, :, :]
    r2 = np.sum(d * d, axis=2)
    s = r2 + eps * eps
    H1 = (2 * eps * eps + r2) / (8 * np.pi * s ** 1.5)
    H2 = 1 / (8 * np.pi * s ** 1.5)
    fd = np.einsum("ijc,jc->ij", d, W)
    T = W[None, :, :] * H1[:, :, None] + (fd * H2)[:, :, None] * d
    np.einsum("iic->ic", T)[:] = 0.0
    return T.sum(1)


def test_direct_vs_numpy_and_invariances():
    X, W = KI.particles(150, seed=12)
    d = O.direct(O.STOKESLET, 0.05, X, W)
    assert O.rel_error(_numpy_stokeslet(X, W, 0.05), d) < 1e-13
    p = np.random.default_rng(0).permutation(150)
    dp = O.direct(O.STOKESLET, 0.05, X[p], W[p])
    assert O.rel_error(d[p], dp) < 1e-14
    assert np.array_equal(O.direct(O.STOKESLET, 0.05, X, np.zeros_like(W)), np.zeros_like(W))
    # targets subset == rows of the full result
    tg = np.array([3, 77, 149])
    assert np.array_equal(O.direct(O.STOKESLET, 0.05, X, W, targets=tg), d[tg])


def test_relative_error_closed_forms(golden):
    for case in golden("worked_examples.json")["relative_error"]["cases"]:
        assert O.rel_error(np.array(case["ref"], float), np.array(case["approx"], float)) == case["E"]


def test_sample_targets_match_full():
    X, W = KI.particles(2000, seed=3)
    T = O.Tree(X, 150)
    F = T.modified_weights(W, 4)
    full = T.treecode(O.STOKESLET, 0.01, 4, 0.7, W, fhat=F)
    tg = KI.sample_targets(2000, 37)
    assert np.array_equal(T.treecode(O.STOKESLET, 0.01, 4, 0.7, W, fhat=F, targets=tg), full[tg])
