"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Gates (BASELINE.json north_star): tree / permutation bit-exact; GPU direct vs
oracle direct relative 2-norm <= 1e-12; GPU treecode vs oracle treecode at
the same tree, n, theta <= 1e-10; per-target interaction counts equal
(integers).  Parity metric = Eq. error with the oracle as the reference.
"""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DIRECT_GATE = 1e-12
TREE_GATE = 1e-10


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1902_02250_b200 import kitc
    return kitc


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def fhat_to_oracle(F, n, pad_zero=True):
    """GPU fhat [C][r][k3][m][j] (row = k1 (n+1) + k2 = 8 r + j, include/kitc.h)
    -> oracle [C][m][(k1 (n+1) + k2) (n+1) + k3].  Checks the padding rows are 0."""
    P = n + 1
    R = (P * P + 7) // 8
    C = F.shape[0]
    m = F.size // (C * R * P * 8)
    G = F.reshape(C, R, P, m, 8).transpose(0, 3, 1, 4, 2).reshape(C, m, R * 8, P)
    if pad_zero:
        assert not G[:, :, P * P:, :].any(), "fhat padding rows must be written as 0"
    return np.ascontiguousarray(G[:, :, : P * P, :]).reshape(C, m, P ** 3)


# ---------------------------------------------------------------- direct sum
@pytest.mark.parametrize("N,kern,eps,self_omit", [
    (1000, 0, 0.01, True), (4099, 0, 0.01, True), (4099, 1, 0.01, True), (3001, 2, 0.05, True),
    (1500, 0, 0.02, False), (1, 0, 1.0, False), (2, 1, 0.01, True), (257, 0, 0.0, True)])
def test_direct_parity(K, N, kern, eps, self_omit):
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, seed=N, m=m)
    ref = O.direct(kern, eps, X, W, self_omit=self_omit)
    got = host(K.direct(dev(X), dev(W), kern, eps, self_omit=self_omit))
    if np.all(ref == 0):
        assert np.all(got == 0)
    else:
        assert O.rel_error(ref, got) <= DIRECT_GATE


# ---------------------------------------------------------------- tree
def assert_same_tree(T, G):
    assert T.nclusters == len(G["begin"])
    assert np.array_equal(T.perm, G["perm"])
    for k in ("begin", "end", "level", "parent", "first_child", "nchild"):
        assert np.array_equal(getattr(T, k), G[k]), k
    assert np.array_equal(T.lo, G["lo"]) and np.array_equal(T.hi, G["hi"])


@pytest.mark.parametrize("N,N0,geom", [(1000, 100, "uniform"), (100_000, 500, "uniform"),
                                       (50_000, 64, "sphere"), (20_000, 40, "slab"),
                                       (5000, 1, "uniform"), (33, 100, "uniform"), (5436, 40, "rods"),
                                       (20000, 100, "organisms")])
def test_tree_bit_exact(K, N, N0, geom):
    X, _ = KI.particles(N, geom, seed=7)
    T = O.Tree(X, N0)
    G = K.Tree(dev(X), N0)
    assert (G.nclusters, G.depth, G.ndegenerate) == (T.nclusters, T.depth, T.ndegenerate)
    assert_same_tree(T, G.export())


def test_tree_degenerate_inputs(K):
    cases = [np.zeros((10, 3)),
             np.array([[0, 0, 0]] * 3 + [[1, 1, 1]] * 3, float),
             np.array([[1.0, 0, 0], [np.nextafter(1.0, 2.0), 0, 0], [np.nextafter(1.0, 2.0), 0, 0]]),
             np.array([[i, j, k] for k in (0, 1) for j in (0, 1) for i in (0, 1)], float)]
    for X in cases:
        T = O.Tree(X, 1)
        G = K.Tree(dev(X), 1)
        assert G.ndegenerate == T.ndegenerate
        assert_same_tree(T, G.export())
    with pytest.raises(K.KitcError) as e:
        K.Tree(dev(np.array([[0.0, np.inf, 0.0], [1.0, 1.0, 1.0]])), 1)
    assert e.value.status == K.KITC_EINVAL


# ---------------------------------------------------------------- weights
@pytest.mark.parametrize("N,N0,n,kern,geom", [(1000, 100, 4, 0, "uniform"), (20_000, 500, 8, 0, "uniform"),
                                              (12_000, 50, 3, 2, "sphere"), (9000, 2000, 10, 1, "uniform")])
def test_modified_weights_parity(K, N, N0, n, kern, geom):
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=3, m=m)
    T = O.Tree(X, N0)
    ref = T.modified_weights(W, n)
    G = K.Tree(dev(X), N0)
    got = fhat_to_oracle(host(G.modified_weights(kern, n, dev(W))), n)
    for c in range(T.nclusters):
        nrm = np.linalg.norm(ref[c])
        assert np.linalg.norm(got[c] - ref[c]) <= 1e-13 * max(nrm, 1e-300), c


# ---------------------------------------------------------------- treecode
def run_gpu(K, X, W, kern, n, theta, N0, eps, self_omit=True):
    G = K.Tree(dev(X), N0)
    fh = G.modified_weights(kern, n, dev(W))
    out, st = G.eval(kern, n, theta, eps, fh, self_omit=self_omit, stats=True)
    return host(out), host(st), G


@pytest.mark.parametrize("N,N0,n,theta,kern,eps,geom", [
    (1000, 100, 4, 0.7, 0, 0.01, "uniform"),      # C1
    (8000, 200, 8, 0.7, 0, 0.01, "uniform"),
    (8000, 200, 8, 0.7, 1, 0.01, "uniform"),      # rotlet
    (6000, 100, 5, 0.6, 2, 0.05, "uniform"),      # Stokeslet + rotlet
    (15000, 300, 6, 0.7, 0, 0.005, "sphere"),
    (7000, 80, 3, 0.5, 0, 0.01, "slab"),
    (3000, 30, 12, 0.7, 0, 0.01, "uniform"),      # generic (runtime-P) kernel
    (600, 20, 2, 0.0, 0, 0.01, "uniform"),        # theta = 0 -> direct
    (2999, 37, 4, 0.7, 0, 0.01, "uniform"),       # odd N, odd leaf bounds: pad source at index N
    (1001, 19, 7, 0.7, 1, 0.02, "sphere"),        # odd N, rotlet, partial last fhat block
    (3, 1, 1, 0.7, 0, 0.01, "uniform"),           # tiny: one-particle leaves
    (3775, 100, 7, 0.7, 2, 0.3, "rods"),          # paper Example 2 geometry (5^2 rods), Stokeslet + rotlet
    (12000, 300, 7, 0.7, 0, 0.02, "organisms"),   # paper Example 1 geometry (organism pairs)
    (4000, 100, 5, 0.7, 0, 0.0, "uniform"),       # eps = 0: the singular (classical) Stokeslet
    (1500, 40, 16, 0.7, 1, 0.01, "uniform"),      # maximum degree n = 16 (runtime-P kernel), rotlet
    (2500, 80, 6, 0.95, 2, 0.02, "slab"),         # theta close to 1, combined kernel, 4-way splits
    (20000, 300, 7, 0.7, 0, 0.01, "uniform"),     # P = 8: far field blocked over target pairs
    (12001, 250, 9, 0.6, 0, 0.01, "uniform"),     # P = 10: the same, odd N
])
def test_treecode_parity(K, N, N0, n, theta, kern, eps, geom):
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=11, m=m)
    T = O.Tree(X, N0)
    ref, rst = T.treecode(kern, eps, n, theta, W, stats=True)
    got, gst, _ = run_gpu(K, X, W, kern, n, theta, N0, eps)
    assert O.rel_error(ref, got) <= TREE_GATE
    assert np.array_equal(rst.astype(np.int64), gst)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7])
def test_far_small_every_degree(K, n):
    # eval.cu far_small (Stokeslet, P = n + 1 <= 8: the whole cluster in one stage, row groups of
    # 1 / 2 / 3 chains, leftover rows pair by pair) with the accepting masks that occur naturally
    # (all 4 targets, 3 of 4 through far_small; 1 or 2 through the team path): many small clusters
    # so partial masks are frequent; sources as targets and separate targets
    X, W = KI.particles(6000, "sphere", seed=20 + n)
    T = O.Tree(X, 40)
    ref, rst = T.treecode(0, 0.02, n, 0.8, W, stats=True)
    got, gst, G = run_gpu(K, X, W, 0, n, 0.8, 40, 0.02)
    assert O.rel_error(ref, got) <= TREE_GATE, n
    assert np.array_equal(rst.astype(np.int64), gst)
    Xt = np.random.default_rng(n).uniform(-1.2, 1.2, (700, 3))
    reft = T.treecode_targets(0, 0.02, n, 0.8, W, Xt)
    fh = G.modified_weights(0, n, dev(W))
    gott = host(G.eval_targets(0, n, 0.8, 0.02, fh, dev(Xt)))
    assert O.rel_error(reft, gott) <= TREE_GATE, n


def test_treecode_self_include(K):
    X, W = KI.particles(4000, seed=2)
    T = O.Tree(X, 150)
    ref = T.treecode(0, 0.02, 6, 0.7, W, self_omit=False)
    got, _, _ = run_gpu(K, X, W, 0, 6, 0.7, 150, 0.02, self_omit=False)
    assert O.rel_error(ref, got) <= TREE_GATE


def test_error_tracks_oracle_vs_n(K):
    # E_gpu(n) tracks E_oracle(n) (north_star): same decisions, rounding-level diffs
    X, W = KI.particles(5000, seed=0)
    d_or = O.direct(0, 0.01, X, W)
    d_gpu = host(K.direct(dev(X), dev(W), 0, 0.01))
    T = O.Tree(X, 250)
    for n in range(1, 11):
        e_or = O.rel_error(d_or, T.treecode(0, 0.01, n, 0.7, W))
        got, _, _ = run_gpu(K, X, W, 0, n, 0.7, 250, 0.01)
        e_gpu = O.rel_error(d_gpu, got)
        assert abs(e_gpu - e_or) <= 1e-9 * max(e_or, 1e-16) + 1e-12


def test_split_ranges_bitwise_identical(K):
    # the multi-GPU decomposition (cluster shards + batch shards) is result-invariant
    X, W = KI.particles(30000, seed=5)
    G = K.Tree(dev(X), 400)
    full = G.modified_weights(0, 6, dev(W))
    out_full = G.eval(0, 6, 0.7, 0.01, full)
    parts = torch.zeros_like(full)
    C = G.nclusters
    for cb, ce in [(0, C // 3), (C // 3, C // 2), (C // 2, C)]:
        G.modified_weights(0, 6, dev(W), cluster_range=(cb, ce), fhat=parts)
    assert torch.equal(parts, full)
    out = torch.zeros_like(out_full)
    nb = G.nbatches
    for bb, be in [(0, 17), (17, nb // 2), (nb // 2, nb)]:
        G.eval(0, 6, 0.7, 0.01, parts, out=out, batch_range=(bb, be))
    assert torch.equal(out, out_full)
    # interleaved multi-GPU split (kitc_eval_part): the parts together are bitwise the full run
    for k in (2, 3, 8):
        outp = torch.zeros_like(out_full)
        for r in range(k):
            G.eval(0, 6, 0.7, 0.01, parts, out=outp, part=(r, k))
        assert torch.equal(outp, out_full)
    # run-to-run determinism
    G2 = K.Tree(dev(X), 400)
    assert torch.equal(G2.eval(0, 6, 0.7, 0.01, G2.modified_weights(0, 6, dev(W))), out_full)


def test_state_errors(K):
    X, W = KI.particles(500, seed=1)
    G = K.Tree(dev(X), 50)
    fh = torch.zeros(G.fhat_shape(0, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(K.KitcError) as e:
        G.eval(0, 4, 0.7, 0.01, fh)                          # weights not computed
    assert e.value.status == K.KITC_ESTATE
    G.modified_weights(0, 4, dev(W), fhat=fh)
    with pytest.raises(K.KitcError) as e:                    # n mismatch (C-ABI state check)
        K.kitc_eval(G.handle, 0, 5, 0.7, 50, 0.01, 0, K._ptr(fh), 0, 1, K._ptr(fh), None, K._stream())
    assert e.value.status == K.KITC_ESTATE
    with pytest.raises(K.KitcError):
        K.kitc_eval(G.handle, 0, 4, 0.7, 51, 0.01, 0, K._ptr(fh), 0, 1, K._ptr(fh), None, K._stream())
    with pytest.raises(K.KitcError):
        G.eval(0, 4, 1.0, 0.01, fh)                          # theta >= 1


def test_batch_targets_prefix(K):
    # kitc_batch_targets(b) = targets in batches [0, b): batches tile the sorted positions leaf by leaf
    X, W = KI.particles(7001, seed=8)
    G = K.Tree(dev(X), 90)
    nb = G.nbatches
    pre = np.array([G.batch_targets(b) for b in range(nb + 1)])
    assert pre[0] == 0 and pre[-1] == 7001
    d = np.diff(pre)
    assert d.min() >= 1 and d.max() <= 4
    fh = G.modified_weights(0, 3, dev(W))
    b0, b1 = nb // 3, 2 * nb // 3
    _, st = G.eval(0, 3, 0.7, 0.01, fh, batch_range=(b0, b1), stats=True)
    assert int((host(st)[:, 4] > 0).sum()) == pre[b1] - pre[b0]


def test_treecode_degenerate_inputs(K):
    # coincident / duplicated / lattice points: degenerate leaves (count > N0), zero-size clusters
    # accepted through their (n,n,n) proxy (reading A14), coincident non-self pairs at s = eps^2
    rng = np.random.default_rng(4)
    cases = [np.zeros((10, 3)),
             np.array([[0, 0, 0]] * 30 + [[1, 1, 1]] * 30 + [[0.5, 0.2, 0.9]] * 5, float),
             np.array([[i, j, k] for k in range(4) for j in range(4) for i in range(4)], float),
             np.repeat(rng.uniform(-1, 1, (40, 3)), 7, axis=0)]
    for X in cases:
        W = rng.uniform(-1, 1, (X.shape[0], 3))
        for self_omit in (True, False):
            T = O.Tree(X, 3)
            ref, rst = T.treecode(0, 0.05, 4, 0.7, W, self_omit=self_omit, stats=True)
            got, gst, _ = run_gpu(K, X, W, 0, 4, 0.7, 3, 0.05, self_omit=self_omit)
            assert np.array_equal(rst.astype(np.int64), gst)
            if np.any(ref != 0):
                assert O.rel_error(ref, got) <= TREE_GATE


# ---------------------------------------------------------------- E (A10) and the boundary
@pytest.mark.parametrize("rows,p", [(1, 3), (7, 6), (1000, 3), (1_000_000, 6), (3_333_334, 3)])
def test_rel_error_parity(K, rows, p):
    # kitc_rel_error vs the oracle's orc_rel_error (Eq. error) on the same arrays
    rng = np.random.default_rng(rows)
    ref = rng.standard_normal((rows, p))
    ap = ref * (1.0 + 1e-6 * rng.standard_normal((rows, p)))
    E_or = O.rel_error(ref, ap)
    E_gpu = K.rel_error(dev(ref), dev(ap))
    assert abs(E_gpu - E_or) <= 1e-13 * E_or
    assert K.rel_error(dev(ref), dev(ref)) == 0.0


def test_rel_error_worked_examples(K, golden):
    # the closed forms pinned for the oracle (tests/golden/worked_examples.json) hold for the GPU too
    assert K.rel_error(dev(np.array([[1.0, 0.0, 0.0]])), dev(np.zeros((1, 3)))) == 1.0
    assert abs(K.rel_error(dev(np.array([[3.0, 4.0]])), dev(np.array([[3.0, 0.0]]))) - 0.8) <= 1e-16
    with pytest.raises(K.KitcError) as e:
        K.rel_error(dev(np.zeros((4, 3))), dev(np.ones((4, 3))))
    assert e.value.status == K.KITC_EINVAL
    sc = torch.empty(K.REL_ERROR_SCRATCH, dtype=torch.float64, device="cuda")
    a = dev(np.ones((4, 3)))
    with pytest.raises(K.KitcError):   # NULL scratch
        K.kitc_rel_error(K._ptr(a), K._ptr(a), 12, None, K._stream())
    assert K.kitc_rel_error(K._ptr(a), K._ptr(a), 12, K._ptr(sc), K._stream()) == 0.0


def test_tree_memory_from_torch_allocator(K):
    # the handle's device memory comes from PyTorch's caching allocator (kitc_allocator)
    X, W = KI.particles(50_000, seed=9)
    Xd, Wd = dev(X), dev(W)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    G = K.Tree(Xd, 500)
    G.modified_weights(0, 6, Wd)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - before
    assert held >= 50_000 * 8 * 3 * 2          # at least the sorted coordinates + partition scratch
    G.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - before <= 0


def test_allocator_failure_is_enomem(K):
    import ctypes as C
    fail = K.KitcAllocator(K._ALLOC_FN(lambda n, s, c: None), K._RELEASE_FN(lambda p, s, c: None), None)
    h = K.kitc_tree_create_with_allocator(fail)
    X = dev(KI.particles(1000, seed=1)[0])
    try:
        with pytest.raises(K.KitcError) as e:
            K.kitc_build_tree(h, K._ptr(X), 1000, 100, K._stream())
        assert e.value.status == K.KITC_ENOMEM
    finally:
        K.kitc_tree_free(h)
    bad = K.KitcAllocator(K._ALLOC_FN(lambda n, s, c: None), K._RELEASE_FN(), None)   # NULL release
    hh = C.c_void_p()
    assert K.lib().kitc_tree_create_with_allocator(C.byref(bad), C.byref(hh)) == K.KITC_EINVAL


def test_workspace_bound_covers_the_handle(K):
    # the device memory a handle takes from its allocator stays within kitc_tree_workspace_bytes
    for N, N0, geom in ((200_000, 500, "uniform"), (30_000, 1, "sphere")):
        X, W = KI.particles(N, geom, seed=4)
        Xd, Wd = dev(X), dev(W)
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated()
        G = K.Tree(Xd, N0)
        G.modified_weights(0, 8, Wd)
        torch.cuda.synchronize()
        held = torch.cuda.memory_allocated() - before
        assert 0 < held <= K.kitc_tree_workspace_bytes(N, N0, 0, 8)
        G.close()


# ---------------------------------------------------------------- f4: upward pass for fhat
@pytest.mark.parametrize("N,N0,n,kern,geom", [(20_000, 100, 8, 0, "uniform"), (12_000, 60, 4, 1, "sphere"),
                                              (5436, 50, 6, 2, "rods"), (6000, 30, 3, 0, "slab"),
                                              (3000, 40, 16, 1, "uniform"), (40, 1, 2, 0, "uniform")])
def test_upward_weights_parity(K, N, N0, n, kern, geom):
    # KITC_WEIGHTS_UPWARD vs the oracle's upward pass (<= 1e-13) and vs the direct Algorithm 1 (<= 1e-12)
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=13, m=m)
    T = O.Tree(X, N0)
    U = T.modified_weights(W, n, upward=True)
    D = T.modified_weights(W, n)
    G = K.Tree(dev(X), N0)
    Wd = dev(W)
    got = fhat_to_oracle(host(G.modified_weights(kern, n, Wd, upward=True)), n)
    for c in range(T.nclusters):
        nu = np.linalg.norm(U[c])
        assert np.linalg.norm(got[c] - U[c]) <= 1e-13 * max(nu, 1e-300), c
        assert np.linalg.norm(got[c] - D[c]) <= 1e-12 * max(np.linalg.norm(D[c]), 1e-300), c
    # suffix range (the bench's [1, C)): the same values, the root untouched
    fh = torch.zeros(G.fhat_shape(kern, n), dtype=torch.float64, device="cuda")
    G.modified_weights(kern, n, Wd, cluster_range=(1, G.nclusters), fhat=fh, upward=True)
    g2 = fhat_to_oracle(host(fh), n)
    assert np.array_equal(g2[1:], got[1:]) and not g2[0].any()
    # the treecode with the upward fhat meets the oracle treecode (direct fhat) gate
    out, st = G.eval(kern, n, 0.7, 0.01, G.modified_weights(kern, n, Wd, upward=True), stats=True)
    ref, rst = T.treecode(kern, 0.01, n, 0.7, W, fhat=D, stats=True)
    assert O.rel_error(ref, host(out)) <= 1e-10
    assert np.array_equal(rst.astype(np.int64), host(st))


def test_upward_range_rules(K):
    X, W = KI.particles(5000, seed=2)
    G = K.Tree(dev(X), 100)
    fh = torch.zeros(G.fhat_shape(0, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(K.KitcError) as e:   # children of computed clusters must be in range
        G.modified_weights(0, 4, dev(W), cluster_range=(0, G.nclusters - 1), fhat=fh, upward=True)
    assert e.value.status == K.KITC_EINVAL
    with pytest.raises(K.KitcError):        # unknown flag bits
        K._call("kitc_modified_weights_ex", G.handle, 0, 4, K._ptr(dev(W)), 0, G.nclusters,
                K.C.c_uint32(2), K._ptr(fh), K._stream())


def test_eval_into_pinned_host_output(K):
    # kitc_eval may write its rows straight into pinned host memory (zero-copy): identical values
    X, W = KI.particles(30_000, seed=6)
    G = K.Tree(dev(X), 300)
    fh = G.modified_weights(0, 6, dev(W))
    ref = host(G.eval(0, 6, 0.7, 0.01, fh))
    outh = torch.zeros((30_000, 3), dtype=torch.float64).pin_memory()
    G.eval(0, 6, 0.7, 0.01, fh, out=outh)
    torch.cuda.synchronize()
    assert np.array_equal(outh.numpy(), ref)
    with pytest.raises(ValueError):          # pageable host memory is refused by the binding
        G.eval(0, 6, 0.7, 0.01, fh, out=torch.zeros((30_000, 3), dtype=torch.float64))
