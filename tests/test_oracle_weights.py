"""Oracle pins: modified weights, Algorithm 1.

Pins:
  * moment identities -- for every monomial q = y1^a y2^b y3^c with a,b,c <= n,
    sum_k fhat_k q(s_k) = sum_j f_j q(y_j) (tensor interpolation reproduces
    these exactly; the (n+1)^3 conditions determine fhat uniquely);
  * brute force: fhat from the product-form Lagrange polynomials (Eq.
    Lagrange_polynomial) in 50-digit mpmath;
  * the worked n = 1 example, node hits (flag path), single-particle cluster
    (reading A14), zero / linear weights.
"""
import mpmath as mp
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O


def _fhat(Y, F, n, lo=None, hi=None):
    lo = Y.min(0) if lo is None else np.asarray(lo, float)
    hi = Y.max(0) if hi is None else np.asarray(hi, float)
    return O.modified_weights_box(Y, F, n, lo, hi), lo, hi


@pytest.mark.parametrize("n", [1, 2, 4, 7, 8])
def test_moment_identities(n):
    rng = np.random.default_rng(n)
    Y = rng.uniform([0.1, -0.5, 2.0], [0.6, 0.5, 2.25], (60, 3))
    F = rng.uniform(-1, 1, (60, 1))
    fh, lo, hi = _fhat(Y, F, n)
    fh = fh[0]
    c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
    S = [O.grid(n, lo[l], hi[l]) for l in range(3)]
    # scaled monomials ((y-c)/h)^a keep the identities well conditioned
    U = [(S[l] - c[l]) / h[l] for l in range(3)]
    V = (Y - c) / h
    for a in range(n + 1):
        for b in range(n + 1):
            for cc in range(n + 1):
                lhs = np.einsum("ijk,i,j,k->", fh, U[0] ** a, U[1] ** b, U[2] ** cc)
                rhs = np.sum(F[:, 0] * V[:, 0] ** a * V[:, 1] ** b * V[:, 2] ** cc)
                assert abs(lhs - rhs) < 1e-12 * max(1.0, np.abs(F).sum())


@pytest.mark.parametrize("n", [2, 6])
def test_brute_force_product_form(n):
    mp.mp.dps = 50
    rng = np.random.default_rng(100 + n)
    Y = rng.uniform(-1, 1, (12, 3)) * [0.3, 0.2, 0.1] + [1.0, -2.0, 0.5]
    F = rng.uniform(-1, 1, (12, 3))
    fh, lo, hi = _fhat(Y, F, n)
    S = [O.grid(n, lo[l], hi[l]) for l in range(3)]

    def L(l, k, t):
        s = S[l]
        num = mp.fprod(mp.mpf(t) - mp.mpf(s[j]) for j in range(n + 1) if j != k)
        den = mp.fprod(mp.mpf(s[k]) - mp.mpf(s[j]) for j in range(n + 1) if j != k)
        return num / den

    Lv = [[[L(l, k, Y[j, l]) for k in range(n + 1)] for l in range(3)] for j in range(len(Y))]
    for k1 in range(n + 1):
        for k2 in range(n + 1):
            for k3 in range(n + 1):
                for m in range(3):
                    ref = mp.fsum(Lv[j][0][k1] * Lv[j][1][k2] * Lv[j][2][k3] * F[j, m] for j in range(len(Y)))
                    assert abs(fh[m, k1, k2, k3] - float(ref)) < 1e-12


def test_worked_trilinear(golden):
    g = golden("worked_examples.json")["trilinear_n1"]
    fh, _, _ = _fhat(np.array(g["y"], float), np.array(g["f"], float)[:, None], 1, g["lo"], g["hi"])
    expect = np.zeros((2, 2, 2))
    for k, v in g["fhat_nonzero"].items():
        expect[tuple(int(i) for i in k.split(","))] = v
    assert np.allclose(fh[0], expect, rtol=0, atol=1e-16)


def test_particle_on_node_and_single_particle_cluster():
    n = 4
    lo, hi = np.array([0.0, 0.0, 0.0]), np.array([1.0, 2.0, 4.0])
    S = [O.grid(n, lo[l], hi[l]) for l in range(3)]
    # particle at s_(2,0,1) plus a zero-weight particle spanning the box
    Y = np.array([[S[0][2], S[1][0], S[2][1]], lo, hi])
    F = np.array([[2.5], [0.0], [0.0]])
    fh, _, _ = _fhat(Y, F, n, lo, hi)
    e = np.zeros((n + 1,) * 3)
    e[2, 0, 1] = 2.5
    assert np.array_equal(fh[0], e)
    # single-particle cluster: zero-width box, every node coincides, last k = n
    # wins (reading A14) -> all weight at (n, n, n)
    y = np.array([[0.3, -0.2, 0.7]])
    fh, _, _ = _fhat(y, np.array([[1.0, -2.0, 3.0]]), n)
    for m, v in enumerate([1.0, -2.0, 3.0]):
        e = np.zeros((n + 1,) * 3)
        e[n, n, n] = v
        assert np.array_equal(fh[m], e)


def test_zero_and_linearity_and_total():
    rng = np.random.default_rng(9)
    Y = rng.uniform(-1, 1, (40, 3))
    F, G = rng.uniform(-1, 1, (40, 3)), rng.uniform(-1, 1, (40, 3))
    n = 5
    assert np.array_equal(_fhat(Y, np.zeros((40, 3)), n)[0], np.zeros((3, 6, 6, 6)))
    a, b = 0.7, -1.3
    lhs = _fhat(Y, a * F + b * G, n)[0]
    rhs = a * _fhat(Y, F, n)[0] + b * _fhat(Y, G, n)[0]
    assert np.max(np.abs(lhs - rhs)) < 1e-13
    assert np.allclose(_fhat(Y, F, n)[0].sum(axis=(1, 2, 3)), F.sum(0), rtol=0, atol=1e-13)


def test_tree_weights_equal_per_cluster_algorithm1():
    X, W = KI.particles(3000, seed=4)
    T = O.Tree(X, 200)
    Fh = T.modified_weights(W, 3)
    Xs, Ws = X[T.perm], W[T.perm]
    for c in range(T.nclusters):
        b, e = T.begin[c], T.end[c]
        ref = O.modified_weights_box(Xs[b:e], Ws[b:e], 3, T.lo[c], T.hi[c]).reshape(3, -1)
        assert np.array_equal(Fh[c], ref)
