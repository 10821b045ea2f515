"""Full-size parity at the BASELINE configs (C3, C4 at n = 8 and n = 4, C5), in
the launch configuration bench.py times (fhat of clusters [1, C) -- the root is
never accepted, reading A16 -- and kitc_eval_part over all batches).

Oracle side: the single-threaded oracle run in worker processes over cluster
ranges / target slices (oracle/par.py; bitwise the serial oracle,
tests/test_oracle_par.py).  Gates (BASELINE.json north_star):
  * tree / permutation bit-exact;
  * GPU fhat vs oracle fhat <= 1e-13 (relative, all clusters);
  * GPU treecode vs oracle treecode on >= 1e4 sampled targets: relative 2-norm
    (Eq. error) <= 1e-10 AND every sampled target's own relative
    error <= 1e-8 (so one wrong target is visible by itself); interaction
    counts integer-equal;
  * GPU direct sum vs oracle direct sum on 1e4 sampled targets <= 1e-12;
  * E(treecode vs direct) of the GPU tracks the oracle's on the same sample
    (|E_gpu - E_oracle| <= 1e-10 + 2e-12, the triangle inequality on the two gates).
Each test appends its measured numbers to gpurun_out/parity_fullsize.jsonl.
"""
import json
import os
import time

import numpy as np
import pytest

import kitc_inputs as KI
import oracle as O
from oracle.par import ParOracle, host_cores

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIRECT_GATE = 1e-12
TREE_GATE = 1e-10
PER_TARGET_GATE = 1e-8
FHAT_GATE = 1e-13


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


def fhat_to_oracle(F, n):
    P = n + 1
    R = (P * P + 7) // 8
    C = F.shape[0]
    m = F.size // (C * R * P * 8)
    G = F.reshape(C, R, P, m, 8).transpose(0, 3, 1, 4, 2).reshape(C, m, R * 8, P)
    assert not G[:, :, P * P:, :].any(), "fhat padding rows must be written as 0"
    return np.ascontiguousarray(G[:, :, : P * P, :]).reshape(C, m, P ** 3)


def per_target_rel(ref, got):
    """max over targets of |got_i - ref_i| / |ref_i| (2-norm over the p components)."""
    d = np.linalg.norm(got - ref, axis=1)
    r = np.linalg.norm(ref, axis=1)
    return float(np.max(d / np.where(r > 0, r, 1.0)))


def report(rec):
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_fullsize.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


def bench_launch(K, X, W, kern, n, theta, N0, eps):
    """The bench's step: build, fhat of clusters [1, C), kitc_eval_part(0, 1) with stats."""
    G = K.Tree(dev(X), N0)
    Wd = dev(W)
    fh = torch.zeros(G.fhat_shape(kern, n), dtype=torch.float64, device="cuda")
    G.modified_weights(kern, n, Wd, cluster_range=(1, G.nclusters), fhat=fh)
    out, st = G.eval(kern, n, theta, eps, fh, part=(0, 1), stats=True)
    return G, Wd, fh, host(out), host(st)


def run_config(K, name, n=None, S_tree=10_000, S_direct=10_000, direct_all_gpu=True):
    c = dict(KI.CONFIGS[name])
    if n is not None:
        c["n"] = n
    kern, n, theta, N0, eps, N = c["kernel"], c["n"], c["theta"], c["N0"], c["eps"], c["N"]
    X, W = KI.config_particles(name)
    t0 = time.time()
    G, Wd, fh, got, gst = bench_launch(K, X, W, kern, n, theta, N0, eps)
    t_gpu = time.time() - t0
    tg = KI.sample_targets(N, S_tree, seed=31)
    td = tg[np.linspace(0, len(tg) - 1, S_direct).astype(np.int64)] if S_direct < len(tg) else tg
    rec = {"config": name, "N": N, "kernel": kern, "n": n, "theta": theta, "eps": eps, "N0": N0,
           "sample_treecode": int(len(tg)), "sample_direct": int(len(td))}
    with ParOracle(X, W, N0, procs=min(host_cores(), 32)) as P:
        rec["oracle_processes"] = P.procs
        T = P.tree
        # tree bit-exact
        assert (G.nclusters, G.depth, G.ndegenerate) == (T.nclusters, T.depth, T.ndegenerate)
        ex = G.export()
        assert np.array_equal(ex["perm"], T.perm)
        for k in ("begin", "end", "level", "parent", "first_child", "nchild"):
            assert np.array_equal(ex[k], getattr(T, k)), k
        assert np.array_equal(ex["lo"], T.lo) and np.array_equal(ex["hi"], T.hi)
        rec["clusters"], rec["depth"] = int(T.nclusters), int(T.depth)
        # modified weights (all clusters but the root, as the bench computes them)
        t0 = time.time()
        F = P.modified_weights(n)
        rec["t_oracle_weights_s"] = time.time() - t0
        Fg = fhat_to_oracle(host(fh), n)
        dF = np.linalg.norm((Fg[1:] - F[1:]).ravel()) / np.linalg.norm(F[1:].ravel())
        rec["fhat_rel"] = float(dF)
        assert dF <= FHAT_GATE
        # f4: the upward pass (KITC_WEIGHTS_UPWARD) against the direct Algorithm 1 fhat
        fu = torch.zeros_like(fh)
        G.modified_weights(kern, n, Wd, cluster_range=(1, G.nclusters), fhat=fu, upward=True)
        Fu = fhat_to_oracle(host(fu), n)
        rec["fhat_upward_rel"] = float(np.linalg.norm((Fu[1:] - F[1:]).ravel()) / np.linalg.norm(F[1:].ravel()))
        assert rec["fhat_upward_rel"] <= 1e-12
        # treecode at the sampled targets
        t0 = time.time()
        ref, rst = P.treecode(kern, eps, n, theta, F, tg, stats=True)
        rec["t_oracle_treecode_s"] = time.time() - t0
        rec["treecode_rel_2norm"] = float(O.rel_error(ref, got[tg]))
        rec["treecode_max_target_rel"] = per_target_rel(ref, got[tg])
        rec["stats_equal"] = bool(np.array_equal(rst.astype(np.int64), gst[tg]))
        rec["pairs_per_target_sample"] = float((rst[:, 1] + rst[:, 3]).mean())
        # every target of the full run covers all N sources exactly once (Σ N_C = N)
        rec["coverage_all_targets"] = bool(np.all(gst[:, 4] == N))
        # direct sum at the direct sample
        t0 = time.time()
        dref = P.direct(kern, eps, td)
        rec["t_oracle_direct_s"] = time.time() - t0
    if direct_all_gpu:
        dgot_all = host(K.direct(dev(X), Wd, kern, eps))
        dgot = dgot_all[td]
    else:
        dgot = host(K.direct_sample(dev(X), Wd, kern, eps, torch.from_numpy(td).cuda()))
    rec["direct_rel_2norm"] = float(O.rel_error(dref, dgot))
    # the method's error on the direct sample, GPU vs oracle (north_star: E_gpu tracks E_oracle)
    pos = np.searchsorted(tg, td)
    rec["E_gpu"] = float(O.rel_error(dgot, got[td]))
    rec["E_oracle"] = float(O.rel_error(dref, ref[pos]))
    rec["t_gpu_s"] = t_gpu
    report(rec)
    assert rec["treecode_rel_2norm"] <= TREE_GATE
    assert rec["treecode_max_target_rel"] <= PER_TARGET_GATE
    assert rec["stats_equal"] and rec["coverage_all_targets"]
    assert rec["direct_rel_2norm"] <= DIRECT_GATE
    # triangle inequality: |E_gpu - E_oracle| <= treecode difference + direct difference (relative)
    assert abs(rec["E_gpu"] - rec["E_oracle"]) <= TREE_GATE + 2 * DIRECT_GATE
    assert 1e-10 < rec["E_gpu"] < 1e-3
    return rec


def test_C3_full_size(K):
    run_config(K, "C3")


def test_C4_full_size_n8(K):
    run_config(K, "C4")


def test_C4_full_size_n4(K):
    # BASELINE config 4 at its other degree, n = 4
    run_config(K, "C4", n=4)


def test_C5_full_size(K):
    # N = 1e7 points on the unit sphere: treecode VALUES on 1e4 sampled targets
    run_config(K, "C5", direct_all_gpu=False)
