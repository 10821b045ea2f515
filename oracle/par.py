"""Process-parallel driver of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/ and bench.py's cpu_baseline / ``--impl reference`` legs may use it
(same rule as the rest of ``oracle/``).  It holds NO arithmetic: the single-
threaded oracle (oracle/kitc_oracle.c) runs unchanged in P worker processes
over disjoint cluster ranges (Algorithm 1) or disjoint
target slices (Algorithm 2; the direct sum).
Each cluster's fhat and each target's sum are computed exactly as in one
process -- the split changes no number, it only makes the full-size parity
tests (N = 1e6, 1e7) finish in seconds.

Workers are started with the "spawn" method (safe after the parent has
initialised CUDA); each loads the inputs from .npy files written once by the
parent and builds its own oracle tree.  fhat lives in POSIX shared memory so
no worker copies it.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import shutil
import tempfile
from multiprocessing import shared_memory

import numpy as np

from . import DIMS, Tree

_W = {}   # worker state: X, W, tree, attached shared fhat


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _init(xpath, wpath, N0):
    X = np.load(xpath, mmap_mode="r")
    _W["X"] = np.ascontiguousarray(X)
    _W["W"] = np.ascontiguousarray(np.load(wpath, mmap_mode="r"))
    _W["T"] = Tree(_W["X"], N0)
    _W["F"] = None


def _attach(name, shape):
    cur = _W.get("F")
    if cur is not None and cur[0].name == name:
        return cur[1]
    if cur is not None:
        cur[0].close()
    shm = shared_memory.SharedMemory(name=name)
    F = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
    _W["F"] = (shm, F)
    return F


def _weights(job):
    name, shape, n, cb, ce = job
    F = _attach(name, shape)
    _W["T"].modified_weights(_W["W"], n, cluster_range=(cb, ce), out=F)
    return ce - cb


def _treecode(job):
    name, shape, kernel, eps, n, theta, tg, self_omit, stats, size_check = job
    F = _attach(name, shape)
    return _W["T"].treecode(kernel, eps, n, theta, _W["W"], fhat=F, targets=tg, self_omit=self_omit,
                            stats=stats, size_check=size_check)


def _direct(job):
    from . import direct
    kernel, eps, tg, self_omit = job
    return direct(kernel, eps, _W["X"], _W["W"], targets=tg, self_omit=self_omit)


class ParOracle:
    """The oracle over X[N,3], W[N,m] with leaf size N0, run in `procs` processes.

    .tree is the parent's own oracle tree (for sizes, ranges and export)."""

    def __init__(self, X, W, N0, procs=None):
        self.procs = max(1, procs or host_cores())
        self.dir = tempfile.mkdtemp(prefix="kitc_par_oracle_")
        xp, wp = os.path.join(self.dir, "X.npy"), os.path.join(self.dir, "W.npy")
        np.save(xp, np.ascontiguousarray(X, dtype=np.float64))
        np.save(wp, np.ascontiguousarray(W, dtype=np.float64))
        self.m = np.asarray(W).reshape(len(X), -1).shape[1]
        self.N0 = int(N0)
        self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_init, initargs=(xp, wp, self.N0))
        self.tree = Tree(X, N0)
        self._shm = []
        self._names = {}

    # -- fhat in shared memory -------------------------------------------------
    def _fhat_buffer(self, n):
        shape = (self.tree.nclusters, self.m, (n + 1) ** 3)
        shm = shared_memory.SharedMemory(create=True, size=max(8, int(np.prod(shape)) * 8))
        self._shm.append(shm)
        F = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
        F[:] = 0.0
        return shm, F

    def modified_weights(self, n):
        """Algorithm 1 for every cluster; returns fhat [C][m][(n+1)^3] in shared memory,
        valid until close() (copy it to keep it)."""
        shm, F = self._fhat_buffer(n)
        sizes = (self.tree.end - self.tree.begin).astype(np.float64)
        cum = np.concatenate([[0.0], np.cumsum(sizes)])
        k = 4 * self.procs   # cluster ranges balanced by sum of N_C (Algorithm 1 costs O(N_C n^3))
        cuts = sorted(set([0] + [int(np.searchsorted(cum, cum[-1] * r / k)) for r in range(1, k)] +
                          [self.tree.nclusters]))
        jobs = [(shm.name, F.shape, n, b, e) for b, e in zip(cuts[:-1], cuts[1:]) if e > b]
        assert sum(self.pool.map(_weights, jobs, chunksize=1)) == self.tree.nclusters
        self._names[F.ctypes.data] = shm.name
        return F

    def _fhat_name(self, F):
        if F.ctypes.data not in self._names:
            raise ValueError("fhat must come from ParOracle.modified_weights (valid until close())")
        return self._names[F.ctypes.data]

    def treecode(self, kernel, eps, n, theta, F, targets, self_omit=True, stats=False, size_check=False):
        """Algorithm 2 at the given target indices (original order), split over the workers."""
        name = self._fhat_name(F)
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        parts = [p for p in np.array_split(tg, 4 * self.procs) if p.size]
        res = self.pool.map(_treecode, [(name, F.shape, kernel, eps, n, theta, p, self_omit, stats, size_check)
                                        for p in parts], chunksize=1)
        if stats:
            return np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res])
        return np.concatenate(res)

    def direct(self, kernel, eps, targets, self_omit=True):
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        parts = [p for p in np.array_split(tg, 4 * self.procs) if p.size]
        return np.concatenate(self.pool.map(_direct, [(kernel, eps, p, self_omit) for p in parts], chunksize=1))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None
        for shm in self._shm:
            for op in (shm.unlink, shm.close):   # close() fails while arrays still view it: unlink first
                try:
                    op()
                except Exception:
                    pass
        self._shm = []
        self._names = {}
        shutil.rmtree(self.dir, ignore_errors=True)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


__all__ = ["ParOracle", "host_cores", "DIMS"]
