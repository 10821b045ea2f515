"""Oracle pins: the upward pass for modified weights (orc_modified_weights_upward,
not in the paper -- SURVEY.md §8(f) f4; reading A24).

An internal cluster's fhat is Algorithm 1 applied to its children's proxy points
carrying the children's fhat.  Pinned by what fixes fhat uniquely, independently
of either implementation:
  * moment identities of every cluster against its OWN particles:
    sum_k fhat_k q(s_k) = sum_{j in C} f_j q(y_j) for all monomials q of degree
    <= n per axis (Eq. modified_weights; these (n+1)^3 conditions
    determine fhat) -- the same identities as the direct Algorithm 1's pins;
  * hence equality with the (separately pinned) direct Algorithm 1 to rounding,
    leaves bitwise (they are Algorithm 1 on particles in both).
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O


@pytest.mark.parametrize("N,N0,n,geom", [(3000, 40, 3, "uniform"), (2500, 30, 5, "sphere"), (2000, 25, 8, "slab")])
def test_upward_moment_identities(N, N0, n, geom):
    X, W = KI.particles(N, geom, seed=N)
    T = O.Tree(X, N0)
    F = T.modified_weights(W, n, upward=True)
    Xs, Ws = X[T.perm], W[T.perm]
    internal = np.where(T.nchild > 0)[0]
    assert len(internal) >= 3 and T.depth >= 2
    for c in internal:
        lo, hi = T.lo[c], T.hi[c]
        ctr, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
        S = [(O.grid(n, lo[l], hi[l]) - ctr[l]) / h[l] for l in range(3)]
        V = (Xs[T.begin[c]:T.end[c]] - ctr) / h
        f = Ws[T.begin[c]:T.end[c]]
        P = n + 1
        fh = F[c].reshape(3, P, P, P)
        for a in range(P):
            for b in range(P):
                for cc in range(P):
                    q = V[:, 0] ** a * V[:, 1] ** b * V[:, 2] ** cc
                    lhs = np.einsum("mijk,i,j,k->m", fh, S[0] ** a, S[1] ** b, S[2] ** cc)
                    rhs = f.T @ q
                    assert np.all(np.abs(lhs - rhs) <= 1e-11 * max(1.0, np.abs(f).sum())), (c, a, b, cc)


@pytest.mark.parametrize("N,N0,n,geom,kern", [(20000, 100, 8, "uniform", 0), (12000, 60, 4, "sphere", 1),
                                               (6000, 50, 6, "rods", 2)])
def test_upward_equals_direct_algorithm1(N, N0, n, geom, kern):
    m = O.DIMS[kern][0]
    if geom == "rods":
        N = 6 * 6 * 151
    X, W = KI.particles(N, geom, seed=3, m=m)
    T = O.Tree(X, N0)
    D = T.modified_weights(W, n)
    U = T.modified_weights(W, n, upward=True)
    leaf = T.nchild == 0
    assert np.array_equal(U[leaf], D[leaf])
    for c in np.where(~leaf)[0]:
        assert np.linalg.norm(U[c] - D[c]) <= 1e-12 * np.linalg.norm(D[c]), c


def test_upward_single_leaf_tree_is_algorithm1():
    X, W = KI.particles(50, seed=1)
    T = O.Tree(X, 100)
    assert T.nclusters == 1
    assert np.array_equal(T.modified_weights(W, 5, upward=True), T.modified_weights(W, 5))
