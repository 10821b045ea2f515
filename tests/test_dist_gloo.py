"""Multi-process host logic of the multi-GPU path (paper_1902_02250_b200/dist.py),
world size 2 over gloo on CPU: cluster / batch sharding and the fhat all-gather
reassembly reproduce the single-process fhat bit for bit.  The fhat data are
the oracle's (test-only), the sharding / exchange code is the product's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import kitc_inputs as KI


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _load_dist():
    import importlib.util
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("kitc_dist", os.path.join(root, "paper_1902_02250_b200", "dist.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules["kitc_dist"] = m
    spec.loader.exec_module(m)
    return m


def test_balanced_ranges():
    D = _load_dist()
    w = np.array([100, 10, 10, 10, 10, 10, 10, 10, 10, 10, 10])
    for k in (1, 2, 3, 4, 8, 16):
        r = D.balanced_ranges(w, k)
        assert len(r) == k and r[0][0] == 0 and r[-1][1] == len(w)
        assert all(r[i][1] == r[i + 1][0] for i in range(k - 1))
        assert all(b <= e for b, e in r)
    r = D.cluster_shards(np.array([0, 0, 5, 7]), np.array([10, 5, 7, 10]), 2, skip_root=True)
    assert r[0][0] == 1                                  # root skipped (reading A16, targets = sources)
    r = D.cluster_shards(np.array([0, 0, 5, 7]), np.array([10, 5, 7, 10]), 2)
    assert r[0][0] == 0 and r[-1][1] == 4                # default: every cluster (separate targets may accept the root)


def _worker(rank, world, port, F, shards_expect, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D = _load_dist()
        C = F.shape[0]
        sizes = np.full(C, 7)
        shards = D.cluster_shards(np.zeros(C), sizes, world, skip_root=False)
        assert shards == shards_expect
        S = D.padded_shard_size(shards)
        gathered = torch.zeros((world, S) + F.shape[1:], dtype=torch.float64)
        cb, ce = shards[rank]
        gathered[rank, : ce - cb] = torch.from_numpy(F[cb:ce])  # "this rank's kernel output"
        full = torch.zeros_like(torch.from_numpy(F))
        D.all_gather_fhat(full, gathered, gathered[rank], shards, rank)
        q.put((rank, bool(torch.equal(full, torch.from_numpy(F)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_fhat_all_gather_world2(world):
    import oracle as O
    X, W = KI.particles(3000, seed=9)
    T = O.Tree(X, 150)
    F = T.modified_weights(W, 3)
    D = _load_dist()
    expect = D.cluster_shards(np.zeros(T.nclusters), np.full(T.nclusters, 7), world, skip_root=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, F, expect, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def test_batch_shards_cover_all_targets():
    D = _load_dist()
    counts = np.array([4, 4, 3, 4, 1, 4, 4, 2, 4, 4])
    prefix = np.concatenate([[0], np.cumsum(counts)])
    for k in (1, 2, 3, 8):
        sh = D.batch_shards(prefix, k)
        assert sh[0][0] == 0 and sh[-1][1] == len(counts)
        assert sum(prefix[e] - prefix[b] for b, e in sh) == counts.sum()
