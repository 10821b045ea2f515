"""Python binding of libkitc.so (include/kitc.h) -- argument marshalling only.

Every step of the KITC path runs in the library's CUDA kernels; this module
passes pointers, sizes and the current CUDA stream through ctypes, and uses
PyTorch only for device memory and streams.  There is NO CPU fallback: if
libkitc.so is missing or fails to load, importing this module raises.

Raw entry points carry the C names (kitc_build_tree, kitc_modified_weights,
kitc_eval, kitc_direct, ...).  `Tree` and `treecode()` are the convenience
layer: `treecode(X, W, kernel, n, theta, N0, eps)` is the one-shot
``eval(kernel, n, theta, N0, eps)`` of the north star, chaining
build_tree -> modified_weights -> eval.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KITC_LIB") or os.path.join(_HERE, "libkitc.so")  # override: tuning builds only

KITC_OK, KITC_EINVAL, KITC_ENOMEM, KITC_ECUDA, KITC_ESTATE = 0, -1, -2, -3, -4
STOKESLET, ROTLET, STOKESLET_ROTLET = 0, 1, 2
SELF_OMIT, SELF_INCLUDE = 0, 1
EVAL_SIZE_CHECK = 1   # kitc_eval_flag (include/kitc.h)
WEIGHTS_UPWARD = 1    # kitc_weights_flag
KERNELS = {"stokeslet": STOKESLET, "rotlet": ROTLET, "stokeslet_rotlet": STOKESLET_ROTLET}

# every symbol include/kitc.h declares
EXPORTS = ("kitc_kernel_dims", "kitc_fhat_cluster_len", "kitc_tree_create", "kitc_tree_create_with_allocator",
           "kitc_tree_workspace_bytes", "kitc_build_tree", "kitc_tree_info",
           "kitc_tree_export", "kitc_modified_weights", "kitc_modified_weights_ex", "kitc_modified_weights_peers", "kitc_eval", "kitc_eval_ex", "kitc_eval_part", "kitc_eval_targets", "kitc_eval_targets_ex", "kitc_batch_targets",
           "kitc_direct", "kitc_direct_sample", "kitc_rel_error", "kitc_tree_free", "kitc_last_error",
           "kitc_launch_count", "kitc_build_flags")


class KitcError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


# kitc_allocator (include/kitc.h): device memory of tree handles from PyTorch's caching allocator
_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_RELEASE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class KitcAllocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("release", _RELEASE_FN), ("ctx", C.c_void_p)]


def _torch_alloc(nbytes, stream, ctx):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0))
    except Exception:   # out of memory -> NULL -> KITC_ENOMEM
        return None


def _torch_release(ptr, stream, ctx):
    torch.cuda.caching_allocator_delete(int(ptr))


TORCH_ALLOCATOR = KitcAllocator(_ALLOC_FN(_torch_alloc), _RELEASE_FN(_torch_release), None)
REL_ERROR_SCRATCH = 1184   # KITC_REL_ERROR_SCRATCH


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libkitc.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    i32, i64, d, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
    P = C.POINTER
    sig = {
        "kitc_kernel_dims": [i32, P(i32), P(i32)],
        "kitc_tree_create": [P(vp)],
        "kitc_tree_create_with_allocator": [P(KitcAllocator), P(vp)],
        "kitc_build_tree": [vp, vp, i64, i32, vp],
        "kitc_tree_workspace_bytes": [i64, i32, i32, i32, P(C.c_size_t)],
        "kitc_tree_info": [vp, P(i64), P(i32), P(i64), P(i32)],
        "kitc_tree_export": [vp] + [vp] * 9,
        "kitc_modified_weights": [vp, i32, i32, vp, i64, i64, vp, vp],
        "kitc_modified_weights_peers": [vp, i32, i32, vp, i64, i64, vp, i32, vp],
        "kitc_modified_weights_ex": [vp, i32, i32, vp, i64, i64, C.c_uint32, vp, vp],
        "kitc_fhat_cluster_len": [i32, i32, P(i64)],
        "kitc_eval": [vp, i32, i32, d, i32, d, i32, vp, i64, i64, vp, vp, vp],
        "kitc_eval_ex": [vp, i32, i32, d, i32, d, i32, C.c_uint32, vp, i64, i64, vp, vp, vp],
        "kitc_eval_part": [vp, i32, i32, d, i32, d, i32, C.c_uint32, vp, i32, i32, vp, vp, vp],
        "kitc_eval_targets": [vp, i32, i32, d, i32, d, vp, vp, i64, vp, vp, vp],
        "kitc_eval_targets_ex": [vp, i32, i32, d, i32, d, C.c_uint32, vp, vp, i64, vp, vp, vp],
        "kitc_batch_targets": [vp, i64, P(i64)],
        "kitc_direct": [i32, d, i32, vp, i64, vp, vp, i64, vp, vp],
        "kitc_direct_sample": [i32, d, i32, vp, i64, vp, vp, i64, vp, vp],
        "kitc_rel_error": [vp, vp, i64, vp, P(d), vp],
        "kitc_tree_free": [vp],
        "kitc_last_error": [],
        "kitc_launch_count": [],
        "kitc_build_flags": [],
    }
    global SIGNATURES
    SIGNATURES = sig
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int32
    L.kitc_tree_free.restype = None
    L.kitc_last_error.restype = C.c_char_p
    L.kitc_launch_count.restype = C.c_uint64
    L.kitc_build_flags.restype = C.c_uint32
    return L


_lib = _load()


def lib():
    return _lib


def _call(name, *args):
    st = getattr(_lib, name)(*args)
    if st != KITC_OK:
        raise KitcError(name, st, _lib.kitc_last_error().decode())
    return st


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dev_f64(t, shape1):
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    if t.dim() != 2 or t.shape[1] != shape1:
        raise ValueError(f"expected shape [N, {shape1}], got {tuple(t.shape)}")
    return t


def _buf_f64(t, numel, what, host_ok=False):
    """A caller-provided buffer the kernels index: contiguous fp64 CUDA (or, host_ok, pinned host
    memory -- mapped into the device address space under unified addressing), exact size."""
    where = t.is_cuda or (host_ok and t.is_pinned())
    if not (where and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{what}: expected a contiguous float64 CUDA tensor" + (" or pinned host tensor" if host_ok else ""))
    if t.numel() != numel:
        raise ValueError(f"{what}: expected {numel} elements, got {t.numel()}")
    return t


# ---- raw C entry points (same names as include/kitc.h) -----------------------

def kitc_kernel_dims(kernel):
    m, p = C.c_int32(), C.c_int32()
    _call("kitc_kernel_dims", int(kernel), C.byref(m), C.byref(p))
    return m.value, p.value


def kitc_fhat_cluster_len(kernel, n):
    ln = C.c_int64()
    _call("kitc_fhat_cluster_len", int(kernel), int(n), C.byref(ln))
    return ln.value


def kitc_tree_create():
    h = C.c_void_p()
    _call("kitc_tree_create", C.byref(h))
    return h


def kitc_tree_create_with_allocator(allocator=None):
    """allocator: a KitcAllocator (default: PyTorch's caching allocator)."""
    h = C.c_void_p()
    _call("kitc_tree_create_with_allocator", C.byref(allocator or TORCH_ALLOCATOR), C.byref(h))
    return h


def kitc_tree_workspace_bytes(N, N0, kernel, n):
    b = C.c_size_t()
    _call("kitc_tree_workspace_bytes", int(N), int(N0), int(kernel), int(n), C.byref(b))
    return b.value


def kitc_build_tree(t, xyz_ptr, N, N0, stream_ptr):
    return _call("kitc_build_tree", t, xyz_ptr, int(N), int(N0), stream_ptr)


def kitc_tree_info(t):
    nc, dep, nb, nd = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int32()
    _call("kitc_tree_info", t, C.byref(nc), C.byref(dep), C.byref(nb), C.byref(nd))
    return nc.value, dep.value, nb.value, nd.value


def kitc_modified_weights(t, kernel, n, w_ptr, cluster_begin, cluster_end, fhat_ptr, stream_ptr):
    return _call("kitc_modified_weights", t, int(kernel), int(n), w_ptr, int(cluster_begin),
                 int(cluster_end), fhat_ptr, stream_ptr)


def kitc_eval(t, kernel, n, theta, N0, eps, self_mode, fhat_ptr, batch_begin, batch_end, out_ptr,
              stats_ptr, stream_ptr):
    return _call("kitc_eval", t, int(kernel), int(n), float(theta), int(N0), float(eps),
                 int(self_mode), fhat_ptr, int(batch_begin), int(batch_end), out_ptr, stats_ptr,
                 stream_ptr)


def kitc_modified_weights_peers(t, kernel, n, w_ptr, cluster_begin, cluster_end, peer_ptrs, stream_ptr):
    """peer_ptrs: sequence of device addresses (int) of the fhat replicas to write."""
    arr = (C.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
    return _call("kitc_modified_weights_peers", t, int(kernel), int(n), w_ptr, int(cluster_begin),
                 int(cluster_end), C.cast(arr, C.c_void_p), len(peer_ptrs), stream_ptr)


def kitc_eval_ex(t, kernel, n, theta, N0, eps, self_mode, flags, fhat_ptr, batch_begin, batch_end, out_ptr,
                 stats_ptr, stream_ptr):
    return _call("kitc_eval_ex", t, int(kernel), int(n), float(theta), int(N0), float(eps), int(self_mode),
                 C.c_uint32(int(flags)), fhat_ptr, int(batch_begin), int(batch_end), out_ptr, stats_ptr, stream_ptr)


def kitc_eval_targets(t, kernel, n, theta, N0, eps, fhat_ptr, xt_ptr, Nt, out_ptr, stats_ptr, stream_ptr):
    return _call("kitc_eval_targets", t, int(kernel), int(n), float(theta), int(N0), float(eps), fhat_ptr,
                 xt_ptr, int(Nt), out_ptr, stats_ptr, stream_ptr)


def kitc_eval_targets_ex(t, kernel, n, theta, N0, eps, flags, fhat_ptr, xt_ptr, Nt, out_ptr, stats_ptr,
                         stream_ptr):
    return _call("kitc_eval_targets_ex", t, int(kernel), int(n), float(theta), int(N0), float(eps),
                 C.c_uint32(int(flags)), fhat_ptr, xt_ptr, int(Nt), out_ptr, stats_ptr, stream_ptr)


def kitc_batch_targets(t, batch_end):
    v = C.c_int64()
    _call("kitc_batch_targets", t, int(batch_end), C.byref(v))
    return v.value


def kitc_direct(kernel, eps, self_mode, xt_ptr, Nt, xs_ptr, ws_ptr, Ns, out_ptr, stream_ptr):
    return _call("kitc_direct", int(kernel), float(eps), int(self_mode), xt_ptr, int(Nt), xs_ptr,
                 ws_ptr, int(Ns), out_ptr, stream_ptr)


def kitc_rel_error(ref_ptr, approx_ptr, count, scratch_ptr, stream_ptr):
    E = C.c_double()
    _call("kitc_rel_error", ref_ptr, approx_ptr, int(count), scratch_ptr, C.byref(E), stream_ptr)
    return E.value


def kitc_launch_count():
    return int(_lib.kitc_launch_count())


def kitc_build_flags():
    """Bit 0 (KITC_BUILD_CHECKS): the loaded library is the verification build."""
    return int(_lib.kitc_build_flags())


def kitc_tree_free(t):
    _lib.kitc_tree_free(t)


# ---- torch convenience layer ---------------------------------------------------

class Tree:
    """A built KITC tree over device particles X[N, 3]; its device memory comes from
    PyTorch's caching allocator (kitc_tree_create_with_allocator)."""

    def __init__(self, X, N0, stream=None):
        self._h = kitc_tree_create_with_allocator()
        self.build(X, N0, stream)

    def build(self, X, N0, stream=None):
        X = _dev_f64(X, 3)
        self.N, self.N0 = X.shape[0], int(N0)
        kitc_build_tree(self._h, _ptr(X), self.N, self.N0, _stream(stream))
        self.nclusters, self.depth, self.nbatches, self.ndegenerate = kitc_tree_info(self._h)
        return self

    @property
    def handle(self):
        return self._h

    def fhat_shape(self, kernel, n):
        """[C][L]: per cluster [round][k3][comp][8 rows] (include/kitc.h)."""
        return (self.nclusters, kitc_fhat_cluster_len(kernel, n))

    def modified_weights(self, kernel, n, W, cluster_range=None, fhat=None, stream=None, upward=False):
        """upward=True: KITC_WEIGHTS_UPWARD (internal clusters from their children's fhat)."""
        m, _ = kitc_kernel_dims(kernel)
        W = _dev_f64(W, m)
        if fhat is None:
            fhat = torch.empty(self.fhat_shape(kernel, n), dtype=torch.float64, device=W.device)
        _buf_f64(fhat, self.nclusters * kitc_fhat_cluster_len(kernel, n), "fhat")
        cb, ce = cluster_range if cluster_range is not None else (0, self.nclusters)
        if upward:
            _call("kitc_modified_weights_ex", self._h, int(kernel), int(n), _ptr(W), int(cb), int(ce),
                  C.c_uint32(WEIGHTS_UPWARD), _ptr(fhat), _stream(stream))
        else:
            kitc_modified_weights(self._h, kernel, n, _ptr(W), cb, ce, _ptr(fhat), _stream(stream))
        return fhat

    def eval(self, kernel, n, theta, eps, fhat, out=None, batch_range=None, self_omit=True,
             stats=False, stream=None, size_check=False, part=None):
        """part=(p, k): interleaved part p of k (kitc_eval_part) instead of a batch range.
        out may be a pinned host tensor: the kernel then writes the rows straight to host memory."""
        _, p = kitc_kernel_dims(kernel)
        _buf_f64(fhat, self.nclusters * kitc_fhat_cluster_len(kernel, n), "fhat")
        dev = fhat.device
        if out is None:
            out = torch.zeros((self.N, p), dtype=torch.float64, device=dev)
        _buf_f64(out, self.N * p, "out", host_ok=True)
        st = torch.zeros((self.N, 5), dtype=torch.int64, device=dev) if stats else None
        if part is not None:
            _call("kitc_eval_part", self._h, int(kernel), int(n), float(theta), self.N0, float(eps),
                  SELF_OMIT if self_omit else SELF_INCLUDE, C.c_uint32(EVAL_SIZE_CHECK if size_check else 0),
                  _ptr(fhat), int(part[0]), int(part[1]), _ptr(out), _ptr(st), _stream(stream))
            return (out, st) if stats else out
        bb, be = batch_range if batch_range is not None else (0, self.nbatches)
        kitc_eval_ex(self._h, kernel, n, theta, self.N0, eps, SELF_OMIT if self_omit else SELF_INCLUDE,
                     EVAL_SIZE_CHECK if size_check else 0, _ptr(fhat), bb, be, _ptr(out), _ptr(st), _stream(stream))
        return (out, st) if stats else out

    def eval_targets(self, kernel, n, theta, eps, fhat, Xt, out=None, stats=False, stream=None, size_check=False):
        """Treecode at a separate target set Xt[Nt, 3] (device fp64); no self term."""
        _, p = kitc_kernel_dims(kernel)
        Xt = _dev_f64(Xt, 3)
        _buf_f64(fhat, self.nclusters * kitc_fhat_cluster_len(kernel, n), "fhat")
        if out is None:
            out = torch.zeros((Xt.shape[0], p), dtype=torch.float64, device=Xt.device)
        _buf_f64(out, Xt.shape[0] * p, "out")
        st = torch.zeros((Xt.shape[0], 5), dtype=torch.int64, device=Xt.device) if stats else None
        kitc_eval_targets_ex(self._h, kernel, n, theta, self.N0, eps, EVAL_SIZE_CHECK if size_check else 0,
                             _ptr(fhat), _ptr(Xt), Xt.shape[0], _ptr(out), _ptr(st), _stream(stream))
        return (out, st) if stats else out

    def batch_targets(self, batch_end):
        return kitc_batch_targets(self._h, batch_end)

    def export(self):
        """Host copy of the structure (numpy) -- parity checks only."""
        import numpy as np
        k, N = self.nclusters, self.N
        a = dict(perm=np.empty(N, np.int64), begin=np.empty(k, np.int64), end=np.empty(k, np.int64),
                 level=np.empty(k, np.int32), parent=np.empty(k, np.int32),
                 first_child=np.empty(k, np.int32), nchild=np.empty(k, np.int32),
                 lo=np.empty((k, 3)), hi=np.empty((k, 3)))
        vp = lambda x: C.c_void_p(x.ctypes.data)
        _call("kitc_tree_export", self._h, *(vp(a[n]) for n in
                                              ("perm", "begin", "end", "level", "parent", "first_child",
                                               "nchild", "lo", "hi")))
        return a

    def export_ranges(self):
        """Host copy of the cluster ranges only (begin, end)."""
        import numpy as np
        k = self.nclusters
        b, e = np.empty(k, np.int64), np.empty(k, np.int64)
        _call("kitc_tree_export", self._h, None, C.c_void_p(b.ctypes.data), C.c_void_p(e.ctypes.data),
              None, None, None, None, None, None)
        return {"begin": b, "end": e}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            kitc_tree_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def direct(X, W, kernel, eps, self_omit=True, targets=None, out=None, stream=None):
    """O(N^2) sum on the GPU. X[N,3], W[N,m] device fp64; targets default = X."""
    m, p = kitc_kernel_dims(kernel)
    X, W = _dev_f64(X, 3), _dev_f64(W, m)
    T = X if targets is None else _dev_f64(targets, 3)
    if out is None:
        out = torch.empty((T.shape[0], p), dtype=torch.float64, device=X.device)
    _buf_f64(out, T.shape[0] * p, "out")
    kitc_direct(kernel, eps, SELF_OMIT if self_omit else SELF_INCLUDE, _ptr(T), T.shape[0], _ptr(X),
                _ptr(W), X.shape[0], _ptr(out), _stream(stream))
    return out


def direct_sample(X, W, kernel, eps, idx, self_omit=True, out=None, stream=None):
    """Direct sum at the sampled targets X[idx] (idx: device int64) over all sources."""
    m, p = kitc_kernel_dims(kernel)
    X, W = _dev_f64(X, 3), _dev_f64(W, m)
    idx = idx.to(device=X.device, dtype=torch.int64).contiguous()
    if out is None:
        out = torch.empty((idx.numel(), p), dtype=torch.float64, device=X.device)
    _buf_f64(out, idx.numel() * p, "out")
    _call("kitc_direct_sample", int(kernel), float(eps), SELF_OMIT if self_omit else SELF_INCLUDE, _ptr(idx),
          idx.numel(), _ptr(X), _ptr(W), X.shape[0], _ptr(out), _stream(stream))
    return out


def rel_error(ref, approx, stream=None):
    """E of Eq. error on the GPU (rows concatenated)."""
    assert ref.shape == approx.shape and ref.is_contiguous() and approx.is_contiguous()
    scratch = torch.empty(REL_ERROR_SCRATCH, dtype=torch.float64, device=ref.device)
    return kitc_rel_error(_ptr(ref), _ptr(approx), ref.numel(), _ptr(scratch), _stream(stream))


def treecode(X, W, kernel, n, theta, N0, eps, self_omit=True, stats=False, stream=None, tree=None):
    """One-shot eval(kernel, n, theta, N0, eps): build tree, modified weights, evaluate.
    Returns out[N, p] (original order) [, stats[N, 5]]."""
    if isinstance(kernel, str):
        kernel = KERNELS[kernel]
    T = tree.build(X, N0, stream) if tree is not None else Tree(X, N0, stream)
    fhat = T.modified_weights(kernel, n, W, stream=stream)
    return T.eval(kernel, n, theta, eps, fhat, self_omit=self_omit, stats=stats, stream=stream)
