"""Oracle pins: adaptive tree (§6; readings A1-A4).

Every internal cluster is re-checked against the rule as the paper states it,
with numpy on the cluster's own particles: minimal box, leaf iff count <= N0,
bisection of the sides > lmax/sqrt(2) at the midpoint, children = the nonempty
octant/quadrant/half groups in ascending code, stable order inside each child.
Plus hand examples (cube corners, slab -> 4 children) and degenerate inputs.
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O

INV_SQRT2 = 0.7071067811865476


def check_tree(T, X):
    N = X.shape[0]
    assert np.array_equal(np.sort(T.perm), np.arange(N))
    Xs = X[T.perm]
    assert T.begin[0] == 0 and T.end[0] == N and T.parent[0] == -1
    leaves = []
    for c in range(T.nclusters):
        b, e = T.begin[c], T.end[c]
        pts = Xs[b:e]
        assert e > b
        # minimal bounding box (reading A3)
        assert np.array_equal(T.lo[c], pts.min(0)) and np.array_equal(T.hi[c], pts.max(0))
        if T.nchild[c] == 0:
            leaves.append((b, e))
            if e - b > T.N0:
                L = T.hi[c] - T.lo[c]
                assert L.max() == 0.0 or T.ndegenerate > 0     # degenerate leaf only
            continue
        assert e - b > T.N0                                   # reading A1
        L = T.hi[c] - T.lo[c]
        split = L > L.max() * INV_SQRT2                        # P:585-587, A2
        mid = 0.5 * (T.lo[c] + T.hi[c])
        code = ((pts >= mid) & split) @ np.array([1, 2, 4])
        # the parent's particles before partition, in their pre-split order, are
        # the children's concatenated; stable partition => per code, the order of
        # original indices equals their order in the parent's range
        kids = range(T.first_child[c], T.first_child[c] + T.nchild[c])
        codes_present = sorted(set(code.tolist()))
        assert T.nchild[c] == len(codes_present) >= 2          # 8/4/2 children, empties dropped
        pos = b
        for k, cc in zip(kids, codes_present):
            assert T.parent[k] == c and T.level[k] == T.level[c] + 1
            assert T.begin[k] == pos
            assert np.all(code[T.begin[k] - b:T.end[k] - b] == cc)
            pos = T.end[k]
        assert pos == e
    # leaves partition [0, N)
    leaves.sort()
    assert leaves[0][0] == 0 and leaves[-1][1] == N
    assert all(leaves[i][1] == leaves[i + 1][0] for i in range(len(leaves) - 1))
    # BFS order: sorted by (level, begin)
    key = list(zip(T.level.tolist(), T.begin.tolist()))
    assert key == sorted(key)


def check_stability(T, X):
    # within each leaf the original indices keep their input order (a sequence of
    # stable partitions of 0..N-1 preserves relative order inside every group)
    for c in range(T.nclusters):
        if T.nchild[c] == 0:
            seg = T.perm[T.begin[c]:T.end[c]]
            assert np.all(np.diff(seg) > 0)


@pytest.mark.parametrize("N,N0,geom", [(1000, 100, "uniform"), (5000, 64, "sphere"), (3000, 50, "slab"),
                                       (2000, 1, "uniform"), (20000, 500, "uniform")])
def test_tree_rule(N, N0, geom):
    X, _ = KI.particles(N, geom, seed=2)
    T = O.Tree(X, N0)
    check_tree(T, X)
    check_stability(T, X)


def test_cube_corners_eight_leaves():
    X = np.array([[i, j, k] for k in (0, 1) for j in (0, 1) for i in (0, 1)], float)
    T = O.Tree(X, 1)
    assert T.nchild[0] == 8 and T.nclusters == 9
    # child code = bx | by<<1 | bz<<2 -> input order already ascending code
    assert np.array_equal(T.perm, np.arange(8))


def test_slab_four_children():
    g = np.linspace(0.0, 4.0, 5)
    X = np.array([[x, y, z] for x in g for y in g for z in (0.0, 1.0)])
    T = O.Tree(X, 1)
    assert T.nchild[0] == 4                                   # 1 < 4/sqrt(2): z not bisected


def test_degenerate_inputs():
    T = O.Tree(np.array([[0.5, 0.5, 0.5]]), 1)
    assert T.nclusters == 1 and T.nchild[0] == 0
    T = O.Tree(np.zeros((10, 3)), 3)                          # coincident: lmax = 0 -> leaf
    assert T.nclusters == 1 and T.ndegenerate == 1
    T = O.Tree(np.array([[0, 0, 0], [1, 0, 0]], float), 1)
    assert T.nclusters == 3 and T.nchild[0] == 2
    # duplicated points: 3 copies of one point + 3 of another, N0 = 1
    X = np.array([[0, 0, 0]] * 3 + [[1, 1, 1]] * 3, float)
    T = O.Tree(X, 1)
    check_tree(T, X)
    assert T.ndegenerate == 2
    with pytest.raises(ValueError):
        O.Tree(np.array([[0, 0, np.nan]]), 1)


def test_adjacent_doubles_degenerate_split():
    # hi = nextafter(lo): the midpoint rounds to lo or hi -> possibly one child
    lo = 1.0
    hi = np.nextafter(1.0, 2.0)
    X = np.array([[lo, 0, 0], [hi, 0, 0], [hi, 0, 0]])
    T = O.Tree(X, 1)
    check_tree(T, X)


def test_depth_and_counts_C2():
    X, _ = KI.particles(100_000)
    T = O.Tree(X, 500)
    check_tree(T, X)
    assert T.depth == 3 and T.nclusters == 585                # 1 + 8 + 64 + 512
