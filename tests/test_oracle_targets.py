"""Oracle pins for the separate-target evaluation (
P:732-733: the targets need not be the sources).  Targets are no sources, so no
self term; the root and any ancestor of a target's position can be accepted.

Pins (each against something other than the function itself):
  * direct_targets vs an independent numpy evaluation of Eq. Velocity_1
     and vs the (pinned) targets = sources direct sum with the self
    term included;
  * theta = 0 -> treecode_targets == direct_targets (only zero-radius clusters
    accepted: exact by reading A14);
  * polynomial test kernel of degree <= n per source coordinate -> far field
    exact -> treecode_targets == direct_targets at theta = 0.7, with targets
    inside and outside the root box (root accepted for the far ones);
  * interaction lists brute-forced in Python at N <= 200 (coverage = N);
  * targets = sources -> identical to the pinned orc_treecode with the self
    term included; far targets: E decays with n.
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O


def _targets(nt, seed, spread=1.5):
    # inside and outside the source cube [-1, 1]^3
    return np.random.default_rng(seed).uniform(-spread, spread, (nt, 3))


def _numpy_stokeslet_targets(X, W, Xt, eps):
    d = Xt[:, None, :] - X[None, :, :]
    r2 = np.sum(d * d, axis=2)
    s = r2 + eps * eps
    H1 = (2 * eps * eps + r2) / (8 * np.pi * s ** 1.5)
    H2 = 1 / (8 * np.pi * s ** 1.5)
    fd = np.einsum("ijc,jc->ij", d, W)
    return (W[None, :, :] * H1[:, :, None] + (fd * H2)[:, :, None] * d).sum(1)


def test_direct_targets_vs_numpy_and_self_include():
    X, W = KI.particles(180, seed=21)
    Xt = _targets(70, 22)
    d = O.direct_targets(O.STOKESLET, 0.03, X, W, Xt)
    assert O.rel_error(_numpy_stokeslet_targets(X, W, Xt, 0.03), d) < 1e-13
    for K in (O.STOKESLET, O.ROTLET, O.STOKESLET_ROTLET):
        m = O.DIMS[K][0]
        X, W = KI.particles(120, seed=23, m=m)
        ds = O.direct_targets(K, 0.02, X, W, X)
        assert np.array_equal(ds, O.direct(K, 0.02, X, W, self_omit=False))


def test_theta_zero_equals_direct_targets():
    for K in (O.STOKESLET, O.ROTLET):
        X, W = KI.particles(400, seed=5)
        Xt = _targets(90, 6)
        T = O.Tree(X, 10)
        d = O.direct_targets(K, 0.01, X, W, Xt)
        for n in (1, 3):
            assert O.rel_error(d, T.treecode_targets(K, 0.01, n, 0.0, W, Xt)) < 1e-13


def test_polynomial_kernel_far_field_exact_targets():
    X, _ = KI.particles(1500, seed=6)
    W = np.random.default_rng(6).uniform(-1, 1, (1500, 1))
    Xt = np.concatenate([_targets(200, 7), _targets(50, 8, spread=6.0)])
    T = O.Tree(X, 40)
    for n in (2, 3, 4):
        u, st = T.treecode_targets(O.POLY, 0.0, n, 0.7, W, Xt, stats=True)
        assert st[:, 0].sum() > 0
        d = O.direct_targets(O.POLY, 0.0, X, W, Xt, poly_deg=n)
        assert O.rel_error(d, u) < 1e-12


def _mac(lo, hi, x, tt):
    c = 0.5 * (lo + hi)
    h = 0.5 * (hi - lo)
    r2 = (h[0] * h[0] + h[1] * h[1]) + h[2] * h[2]
    d = x - c
    R2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
    return R2 > 0.0 and r2 <= tt * R2


@pytest.mark.parametrize("N,N0,theta", [(200, 8, 0.7), (150, 3, 0.5)])
def test_interaction_lists_brute_force_targets(N, N0, theta):
    X, W = KI.particles(N, seed=N0)
    Xt = np.concatenate([_targets(60, N0), _targets(20, N0 + 1, spread=8.0)])
    T = O.Tree(X, N0)
    n = 3
    _, st = T.treecode_targets(O.STOKESLET, 0.01, n, theta, W, Xt, stats=True)
    tt = theta * theta
    anc = {0: []}
    for c in range(1, T.nclusters):
        anc[c] = anc[T.parent[c]] + [T.parent[c]]
    root_accepted = 0
    for i, x in enumerate(Xt):
        macs = [_mac(T.lo[c], T.hi[c], x, tt) for c in range(T.nclusters)]
        far = [c for c in range(T.nclusters) if macs[c] and not any(macs[a] for a in anc[c])]
        near = [c for c in range(T.nclusters) if T.nchild[c] == 0 and not macs[c]
                and not any(macs[a] for a in anc[c])]
        covered = sum(T.end[c] - T.begin[c] for c in far + near)
        near_pairs = sum(T.end[c] - T.begin[c] for c in near)          # no self term
        assert covered == N
        assert list(st[i]) == [len(far), len(far) * (n + 1) ** 3, len(near), near_pairs, covered]
        root_accepted += far == [0]
    assert root_accepted >= 10                                         # far targets: the root alone


def test_targets_equal_sources_matches_self_include():
    X, W = KI.particles(900, seed=31)
    T = O.Tree(X, 40)
    F = T.modified_weights(W, 4)
    a = T.treecode_targets(O.STOKESLET, 0.02, 4, 0.7, W, X, fhat=F)
    b = T.treecode(O.STOKESLET, 0.02, 4, 0.7, W, fhat=F, self_omit=False)
    assert np.array_equal(a, b)


def test_far_targets_error_decays_with_n():
    X, W = KI.particles(2000, seed=41)
    Xt = _targets(100, 42, spread=1.0) * 0.2 + np.array([3.0, 0.0, 0.0])   # a blob at distance 3
    T = O.Tree(X, 100)
    d = O.direct_targets(O.STOKESLET, 0.01, X, W, Xt)
    ns = (2, 4, 6, 8, 10)
    E = [O.rel_error(d, T.treecode_targets(O.STOKESLET, 0.01, n, 0.7, W, Xt)) for n in ns]
    assert all(b < a for a, b in zip(E, E[1:]))
    # only the root is used (r/R ~ 0.6); per source axis the kernel is analytic inside the
    # Bernstein ellipse through the nearest target x = 2.8: rho = 2.8 + sqrt(2.8^2 - 1) = 5.4,
    # i.e. 0.73 decades per degree asymptotically; require > 0.5 over n = 2..10
    slope = -np.polyfit(ns, np.log10(E), 1)[0]
    assert slope > 0.5, slope
