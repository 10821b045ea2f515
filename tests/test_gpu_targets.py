"""GPU parity of the separate-target evaluation (kitc_eval_targets; SURVEY.md
§8(f) row f2) against the oracle's treecode_targets / direct_targets
(tests/test_oracle_targets.py pins them).  Gates as the main parity tests:
treecode <= 1e-10, direct <= 1e-12, interaction counts equal (integers)."""
import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TREE_GATE = 1e-10
DIRECT_GATE = 1e-12


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


def targets(nt, seed, spread=1.5):
    return np.random.default_rng(seed).uniform(-spread, spread, (nt, 3))


@pytest.mark.parametrize("N,N0,n,theta,kern,eps,geom,nt,spread", [
    (8000, 200, 8, 0.7, 0, 0.01, "uniform", 3001, 1.5),    # inside and outside the source box
    (6000, 100, 5, 0.6, 1, 0.02, "uniform", 2000, 3.0),    # rotlet, many exterior targets
    (5000, 150, 4, 0.7, 2, 0.05, "sphere", 1999, 1.2),     # Stokeslet + rotlet, surface sources
    (3000, 40, 12, 0.7, 0, 0.01, "uniform", 777, 1.0),     # generic (runtime-P) kernel
    (2000, 50, 3, 0.0, 0, 0.01, "uniform", 500, 1.0),      # theta = 0 -> direct
    (1000, 30, 6, 0.7, 0, 0.01, "uniform", 5, 50.0),       # ragged batch, far: root accepted
    (1000, 30, 6, 0.7, 0, 0.01, "uniform", 1, 0.5),        # one target
])
def test_eval_targets_parity(K, N, N0, n, theta, kern, eps, geom, nt, spread):
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, geom, seed=13, m=m)
    Xt = targets(nt, 14, spread)
    T = O.Tree(X, N0)
    ref, rst = T.treecode_targets(kern, eps, n, theta, W, Xt, stats=True)
    G = K.Tree(dev(X), N0)
    fh = G.modified_weights(kern, n, dev(W))
    got, gst = G.eval_targets(kern, n, theta, eps, fh, dev(Xt), stats=True)
    assert O.rel_error(ref, host(got)) <= TREE_GATE
    assert np.array_equal(rst.astype(np.int64), host(gst))


def test_eval_targets_equals_self_include_on_sources(K):
    # targets = sources: same interaction lists (integers equal); the sums differ only in
    # rounding order (near-field lane teams depend on the batch-mates)
    X, W = KI.particles(20000, seed=3)
    G = K.Tree(dev(X), 300)
    fh = G.modified_weights(0, 7, dev(W))
    a, sa = G.eval(0, 7, 0.7, 0.01, fh, self_omit=False, stats=True)
    b, sb = G.eval_targets(0, 7, 0.7, 0.01, fh, dev(X), stats=True)
    assert torch.equal(sa, sb)
    assert float((a - b).norm() / a.norm()) < 1e-13


def test_eval_targets_empty_and_errors(K):
    X, W = KI.particles(500, seed=1)
    G = K.Tree(dev(X), 50)
    fh = G.modified_weights(0, 4, dev(W))
    out = G.eval_targets(0, 4, 0.7, 0.01, fh, torch.zeros((0, 3), dtype=torch.float64, device="cuda"))
    assert out.shape == (0, 3)
    xt = dev(targets(10, 0))
    ot = torch.zeros((10, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(K.KitcError):                                 # n mismatch (C-ABI state check)
        K.kitc_eval_targets(G.handle, 0, 5, 0.7, 50, 0.01, K._ptr(fh), K._ptr(xt), 10, K._ptr(ot), None, K._stream())
    with pytest.raises(K.KitcError):
        G.eval_targets(0, 4, 1.0, 0.01, fh, dev(targets(10, 0)))     # theta >= 1


@pytest.mark.parametrize("kern", [0, 1, 2])
def test_direct_targets_parity(K, kern):
    m = O.DIMS[kern][0]
    X, W = KI.particles(3001, seed=17, m=m)
    Xt = targets(999, 18)
    ref = O.direct_targets(kern, 0.01, X, W, Xt)
    got = host(K.direct(dev(X), dev(W), kern, 0.01, self_omit=False, targets=dev(Xt)))
    assert O.rel_error(ref, got) <= DIRECT_GATE


@pytest.mark.parametrize("kern,self_omit", [(0, True), (1, True), (2, False)])
def test_direct_sample_parity(K, kern, self_omit):
    # sampled targets: the oracle's targets= subset with the self term by index
    m = O.DIMS[kern][0]
    X, W = KI.particles(5003, seed=19, m=m)
    tg = KI.sample_targets(5003, 301, seed=2)
    ref = O.direct(kern, 0.01, X, W, targets=tg, self_omit=self_omit)
    got = host(K.direct_sample(dev(X), dev(W), kern, 0.01, torch.from_numpy(tg).cuda(), self_omit=self_omit))
    assert O.rel_error(ref, got) <= DIRECT_GATE
    full = host(K.direct(dev(X), dev(W), kern, 0.01, self_omit=self_omit))
    assert np.array_equal(full[tg], got)          # same per-target arithmetic as the full sum


@pytest.mark.parametrize("N,N0,n,kern", [(20000, 500, 8, 0), (8000, 60, 4, 1), (3000, 10, 6, 2)])
def test_size_check_parity(K, N, N0, n, kern):
    # variant f4: accepted clusters with N_C < (n+1)^3 summed directly (oracle mirrors it)
    m = O.DIMS[kern][0]
    X, W = KI.particles(N, seed=29, m=m)
    T = O.Tree(X, N0)
    ref, rst = T.treecode(kern, 0.01, n, 0.7, W, stats=True, size_check=True)
    G = K.Tree(dev(X), N0)
    fh = G.modified_weights(kern, n, dev(W))
    got, gst = G.eval(kern, n, 0.7, 0.01, fh, stats=True, size_check=True)
    assert O.rel_error(ref, host(got)) <= TREE_GATE
    assert np.array_equal(rst.astype(np.int64), host(gst))
    # separate targets with the variant
    Xt = targets(999, 30)
    ref_t, rst_t = T.treecode_targets(kern, 0.01, n, 0.7, W, Xt, stats=True, size_check=True)
    got_t, gst_t = G.eval_targets(kern, n, 0.7, 0.01, fh, dev(Xt), stats=True, size_check=True)
    assert O.rel_error(ref_t, host(got_t)) <= TREE_GATE
    assert np.array_equal(rst_t.astype(np.int64), host(gst_t))


def test_modified_weights_peers_replicas(K):
    # the fused weights + exchange kernel writes every cluster slice into each replica
    # (here: three local buffers standing in for peer GPUs' mapped buffers)
    X, W = KI.particles(30000, seed=5)
    G = K.Tree(dev(X), 400)
    ref = G.modified_weights(0, 6, dev(W))
    reps = [torch.full_like(ref, float("nan")) for _ in range(3)]
    C = G.nclusters
    for cb, ce in [(0, C // 3), (C // 3, C)]:           # two "ranks"' cluster ranges
        K.kitc_modified_weights_peers(G.handle, 0, 6, K._ptr(dev(W)), cb, ce, [r.data_ptr() for r in reps],
                                      K._stream())
    for r in reps:
        assert torch.equal(r, ref)
    with pytest.raises(K.KitcError):
        K.kitc_modified_weights_peers(G.handle, 0, 6, K._ptr(dev(W)), 0, C, [reps[0].data_ptr()] * 9, K._stream())


def test_peer_fhat_world1(K):
    # dist.PeerFhat (symmetric memory + device barriers) on a one-rank NCCL group
    import os
    import socket
    import torch.distributed as dist
    from paper_1902_02250_b200 import dist as D
    own = not dist.is_initialized()
    if own:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        X, W = KI.particles(20000, seed=6)
        G = K.Tree(dev(X), 300)
        ref = G.modified_weights(0, 5, dev(W))
        pf = D.PeerFhat(G.nclusters, ref.shape[1], torch.device("cuda", 0))
        for _ in range(2):                               # the barriers are reusable across steps
            got = pf.modified_weights(G, 0, 5, dev(W), (0, G.nclusters))
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        assert torch.equal(G.eval(0, 5, 0.7, 0.01, got), G.eval(0, 5, 0.7, 0.01, ref))
    finally:
        if own:
            dist.destroy_process_group()


def test_binding_rejects_wrong_buffers(K):
    # the binding checks the buffers the kernels index (size, dtype, device) before any launch
    X, W = KI.particles(500, seed=1)
    G = K.Tree(dev(X), 50)
    fh = G.modified_weights(0, 4, dev(W))
    with pytest.raises(ValueError):
        G.eval(0, 4, 0.7, 0.01, fh[:-1])                       # short fhat
    with pytest.raises(ValueError):
        G.eval(0, 5, 0.7, 0.01, fh)                            # fhat sized for n = 4
    with pytest.raises(ValueError):
        G.eval(0, 4, 0.7, 0.01, fh, out=torch.zeros((499, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        G.eval_targets(0, 4, 0.7, 0.01, fh.float(), dev(targets(5, 0)))
    with pytest.raises(ValueError):
        K.direct(dev(X), dev(W), 0, 0.01, out=torch.zeros((500, 2), dtype=torch.float64, device="cuda"))
