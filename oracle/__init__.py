"""CPU oracle for the KITC hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_1902_02250_b200) never imports it; the two share no code.

Thin ctypes wrapper around oracle/kitc_oracle.c (plain C, -O2
-ffp-contract=off, single-threaded).  Every numeric step lives in the C file,
which cites the PAPER.md passage each function follows.  Parity status per
function: see DESIGN.md "Oracle pins" (all pinned; the magnitude of E on the
paper's own Example-1 workload is context only, "parity unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kitc_oracle.c")
_LIB = os.path.join(_HERE, "libkitc_oracle.so")

STOKESLET, ROTLET, STOKESLET_ROTLET, POLY = 0, 1, 2, 99
DIMS = {STOKESLET: (3, 3), ROTLET: (3, 6), STOKESLET_ROTLET: (6, 6), POLY: (1, 1)}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c99",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        d, i64, i32, vp = C.c_double, C.c_int64, C.c_int, C.c_void_p
        L.orc_cheb_nodes.argtypes = [i32, vp]
        L.orc_bary_weights.argtypes = [i32, vp]
        L.orc_grid.argtypes = [i32, d, d, vp]
        L.orc_basis.argtypes = [i32, vp, d, vp]
        L.orc_mrs_scalars.argtypes = [d, d, vp]
        L.orc_pair.argtypes = [i32, d, i32, vp, vp, vp, vp]
        L.orc_build_tree.argtypes = [i64, vp, i32, C.POINTER(vp)]
        L.orc_tree_free.argtypes = [vp]
        L.orc_tree_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32)]
        L.orc_tree_export.argtypes = [vp] + [vp] * 9
        L.orc_modified_weights.argtypes = [vp, i32, i32, vp, vp]
        L.orc_modified_weights_range.argtypes = [vp, i32, i32, vp, i64, i64, vp]
        L.orc_modified_weights_box.argtypes = [i64, vp, vp, i32, i32, vp, vp, vp]
        L.orc_modified_weights_upward.argtypes = [vp, i32, i32, vp, vp]
        L.orc_treecode.argtypes = [vp, i32, d, i32, d, i32, vp, vp, vp, i64, vp, vp]
        L.orc_treecode_ex.argtypes = [vp, i32, d, i32, d, i32, i32, vp, vp, vp, i64, vp, vp]
        L.orc_direct.argtypes = [i32, d, i32, i32, i64, vp, vp, vp, i64, vp]
        L.orc_treecode_targets.argtypes = [vp, i32, d, i32, d, i32, vp, vp, vp, i64, vp, vp]
        L.orc_direct_targets.argtypes = [i32, d, i32, i64, vp, vp, vp, i64, vp]
        L.orc_rel_error.argtypes = [vp, vp, i64, i32]
        L.orc_rel_error.restype = d
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def cheb_nodes(n):
    t = np.empty(n + 1)
    lib().orc_cheb_nodes(n, _p(t))
    return t


def bary_weights(n):
    w = np.empty(n + 1)
    lib().orc_bary_weights(n, _p(w))
    return w


def grid(n, lo, hi):
    s = np.empty(n + 1)
    lib().orc_grid(n, float(lo), float(hi), _p(s))
    return s


def basis(n, s, y):
    s = _f64(s)
    L = np.empty(n + 1)
    lib().orc_basis(n, _p(s), float(y), _p(L))
    return L


def mrs_scalars(r, eps):
    o = np.empty(5)
    lib().orc_mrs_scalars(float(r) * float(r), float(eps), _p(o))
    return o


def mrs_scalars_r2(r2, eps):
    o = np.empty(5)
    lib().orc_mrs_scalars(float(r2), float(eps), _p(o))
    return o


def pair(kernel, eps, x, y, f, poly_deg=0):
    m, p = DIMS[kernel]
    x, y, f = _f64(x), _f64(y), _f64(f)
    assert f.size == m
    out = np.empty(p)
    assert lib().orc_pair(kernel, float(eps), poly_deg, _p(x), _p(y), _p(f), _p(out)) == 0
    return out


class Tree:
    """Oracle tree (§6).  Clusters exported in BFS (level, begin) order."""

    def __init__(self, X, N0):
        X = _f64(X).reshape(-1, 3)
        self.N = X.shape[0]
        self.N0 = int(N0)
        h = C.c_void_p()
        rc = lib().orc_build_tree(self.N, _p(X), self.N0, C.byref(h))
        if rc != 0:
            raise ValueError("oracle tree build rejected the input")
        self._h = h
        nc, dep, ndeg = C.c_int64(), C.c_int(), C.c_int()
        lib().orc_tree_info(h, C.byref(nc), C.byref(dep), C.byref(ndeg))
        self.nclusters, self.depth, self.ndegenerate = nc.value, dep.value, ndeg.value
        k = self.nclusters
        self.perm = np.empty(self.N, np.int64)
        self.begin = np.empty(k, np.int64)
        self.end = np.empty(k, np.int64)
        self.level = np.empty(k, np.int32)
        self.parent = np.empty(k, np.int32)
        self.first_child = np.empty(k, np.int32)
        self.nchild = np.empty(k, np.int32)
        self.lo = np.empty((k, 3))
        self.hi = np.empty((k, 3))
        lib().orc_tree_export(h, _p(self.perm), _p(self.begin), _p(self.end), _p(self.level),
                              _p(self.parent), _p(self.first_child), _p(self.nchild),
                              _p(self.lo), _p(self.hi))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_tree_free(h)
            self._h = None

    def modified_weights(self, W, n, cluster_range=None, out=None, upward=False):
        """Algorithm 1 per cluster; upward=True: internal clusters from their children's
        fhat (orc_modified_weights_upward, not in the paper -- SURVEY §8(f) f4)."""
        W = _f64(W)
        m = W.shape[1]
        P = n + 1
        F = np.zeros((self.nclusters, m, P * P * P)) if out is None else out
        if upward:
            assert cluster_range is None
            assert lib().orc_modified_weights_upward(self._h, n, m, _p(W), _p(F)) == 0
        elif cluster_range is None:
            assert lib().orc_modified_weights(self._h, n, m, _p(W), _p(F)) == 0
        else:
            cb, ce = cluster_range
            assert lib().orc_modified_weights_range(self._h, n, m, _p(W), cb, ce, _p(F)) == 0
        return F

    def treecode(self, kernel, eps, n, theta, W, fhat=None, targets=None, self_omit=True,
                 stats=False, size_check=False):
        m, p = DIMS[kernel]
        W = _f64(W).reshape(self.N, m)
        if fhat is None:
            fhat = self.modified_weights(W, n)
        tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
        nt = self.N if tg is None else tg.size
        out = np.empty((nt, p))
        st = np.empty((nt, 5), np.uint64) if stats else None
        rc = lib().orc_treecode_ex(self._h, kernel, float(eps), n, float(theta), int(bool(self_omit)),
                                   int(bool(size_check)), _p(_f64(fhat)), _p(W), _p(tg), nt, _p(out), _p(st))
        assert rc == 0
        return (out, st) if stats else out


    def treecode_targets(self, kernel, eps, n, theta, W, Xt, fhat=None, stats=False, size_check=False):
        """Treecode at a separate target set Xt (nt x 3); no self term."""
        m, p = DIMS[kernel]
        W = _f64(W).reshape(self.N, m)
        Xt = _f64(Xt).reshape(-1, 3)
        if fhat is None:
            fhat = self.modified_weights(W, n)
        nt = Xt.shape[0]
        out = np.empty((nt, p))
        st = np.empty((nt, 5), np.uint64) if stats else None
        rc = lib().orc_treecode_targets(self._h, kernel, float(eps), n, float(theta), int(bool(size_check)),
                                        _p(_f64(fhat)), _p(W),
                                        _p(Xt), nt, _p(out), _p(st))
        assert rc == 0
        return (out, st) if stats else out


def modified_weights_box(Y, Fw, n, lo, hi):
    Y, Fw = _f64(Y).reshape(-1, 3), _f64(Fw)
    Fw = Fw.reshape(Y.shape[0], -1)
    m = Fw.shape[1]
    P = n + 1
    out = np.empty((m, P, P, P))
    lib().orc_modified_weights_box(Y.shape[0], _p(Y), _p(Fw), m, n, _p(_f64(lo)), _p(_f64(hi)),
                                   _p(out))
    return out


def direct(kernel, eps, X, W, targets=None, self_omit=True, poly_deg=0):
    m, p = DIMS[kernel]
    X = _f64(X).reshape(-1, 3)
    N = X.shape[0]
    W = _f64(W).reshape(N, m)
    tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    nt = N if tg is None else tg.size
    out = np.empty((nt, p))
    rc = lib().orc_direct(kernel, float(eps), poly_deg, int(bool(self_omit)), N, _p(X), _p(W),
                          _p(tg), nt, _p(out))
    assert rc == 0
    return out


def direct_targets(kernel, eps, X, W, Xt, poly_deg=0):
    """Direct sum at separate targets Xt (nt x 3) over all sources (no self term)."""
    m, p = DIMS[kernel]
    X = _f64(X).reshape(-1, 3)
    N = X.shape[0]
    W = _f64(W).reshape(N, m)
    Xt = _f64(Xt).reshape(-1, 3)
    out = np.empty((Xt.shape[0], p))
    rc = lib().orc_direct_targets(kernel, float(eps), poly_deg, N, _p(X), _p(W), _p(Xt), Xt.shape[0], _p(out))
    assert rc == 0
    return out


def rel_error(ref, approx):
    ref, approx = _f64(ref), _f64(approx)
    assert ref.shape == approx.shape
    p = ref.shape[1] if ref.ndim == 2 else 1
    return lib().orc_rel_error(_p(ref), _p(approx), ref.size // p, p)
