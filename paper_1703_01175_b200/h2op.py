"""Device-resident H² operator and the reference-facing drop-ins.

`H2Operator` owns one libh2b handle: the packed operator (pack.py) uploaded
once to HBM.  The module-level `matvec` / `matmat_apply` mirror the
reference surface

* ``h2vie.arith.matvec(h2, x)``                    arith.py:108-117
* ``h2vie.arith.matmat_apply(h2, X, col_block)``   arith.py:120-130

(same argument meaning, same ``ValueError`` on a wrong shape, fresh output
arrays, inputs never mutated) and accept either a reference ``H2Matrix``
(packed and uploaded on first use, cached by identity) or a `PackedH2`.

PyTorch is used only for device memory and streams.  There is no CPU path:
construction raises if libh2b.so or an sm_100 device is missing.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _abi
from .pack import PackedH2, pack_h2

_UPLOAD_CHUNK = 1 << 30  # bytes per h2b_upload call


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _torch():
    import torch
    return torch


def _stream_handle(stream):
    if stream is None:
        return C.c_void_p(_torch().cuda.current_stream().cuda_stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


class H2Operator:
    """The operator S (N x N, complex128) resident on one B200.

    Vectors passed to the ``*_perm`` methods are torch complex128 CUDA
    tensors in the cluster-permuted order; `matvec` / `matmat` take and
    return numpy arrays in the original order (the drop-in surface).
    """

    def __init__(self, h2, device=0, _upload=True):
        pk = h2 if isinstance(h2, PackedH2) else pack_h2(h2)
        L = _abi.lib()
        if not L.h2b_device_ok(int(device)):
            raise RuntimeError("no sm_100 (B200) CUDA device visible; the H2 hot path has no CPU "
                               "fallback")
        self.perm = np.asarray(pk.perm)  # not the PackedH2 itself: the cache must not keep it alive
        self.n = pk.n
        self.device = int(device)
        keep = {}

        def arr(name, dtype):
            a = np.ascontiguousarray(getattr(pk, name), dtype=dtype)
            keep[name] = a
            return a

        lay = _abi.Layout()
        lay.n = pk.n
        lay.depth = pk.depth
        lay.num_clusters = pk.num_clusters
        for name in ("level_ptr", "c_start", "c_size", "c_rank", "c_child_lo", "c_child_hi",
                     "c_parent", "s_col", "d_col"):
            setattr(lay, name, _ptr(arr(name, np.int32), C.c_int32))
        for name in ("c_xhat_off", "c_v_off", "c_t_off", "s_row_ptr", "s_off", "d_row_ptr",
                     "d_off", "perm"):
            setattr(lay, name, _ptr(arr(name, np.int64), C.c_int64))
        lay.n_coupling = pk.n_coupling
        lay.n_near = pk.n_near
        far_on_device = ("synthetic" in pk.meta and pk.sbuf.size == 0 and pk.vbuf.size == 0
                         and pk.tbuf.size == 0)
        if far_on_device:
            ev, et, es = pk.far_elems_expected()
        else:
            ev, et, es = int(pk.vbuf.size), int(pk.tbuf.size), int(pk.sbuf.size)
        lay.v_elems, lay.t_elems = ev, et
        near_on_device = pk.dbuf.size == 0 and pk.n_near > 0
        if near_on_device and "geometry" not in pk.meta:
            raise ValueError("operator has no near-field payload and no geometry to assemble it from")
        lay.s_elems, lay.d_elems = es, int(pk.d_elems_expected())
        handle = C.c_void_p()
        _abi.check(L.h2b_create(C.byref(lay), self.device, C.byref(handle)), "h2b_create")
        self._h = handle
        self._finalizer = weakref.finalize(self, L.h2b_destroy, handle)
        if near_on_device:  # near-field sampled in HBM, never uploaded
            from .nearfield import geometry_arrays, self_term
            centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
            diag = k0 ** 2 * self_term(vol, k0)
            centers = np.ascontiguousarray(centers, dtype=np.float64)
            chi = np.ascontiguousarray(chi, dtype=np.complex128)
            _abi.check(L.h2b_assemble_near(handle, centers.ctypes.data, chi.ctypes.data, float(k0),
                                           float(vol), float(diag.real), float(diag.imag)),
                       "h2b_assemble_near")
        if far_on_device:  # structure-exact operator: seeded V/T/S generated in HBM
            from .synthetic import fill_far_field_on_device
            fill_far_field_on_device(L, handle, pk, self.device, pk.meta["synthetic"].get("seed", 0))
        self._lock = threading.Lock()
        self._perm_t = None
        if not _upload:  # tests of the C-ABI's upload bookkeeping upload the payloads themselves
            return
        for sec, buf in ((_abi.SEC_V, pk.vbuf), (_abi.SEC_T, pk.tbuf), (_abi.SEC_S, pk.sbuf),
                         (_abi.SEC_D, pk.dbuf)):
            b = np.ascontiguousarray(buf, dtype=np.complex128).view(np.uint8)
            for off in range(0, b.size, _UPLOAD_CHUNK):
                chunk = b[off:off + _UPLOAD_CHUNK]
                _abi.check(L.h2b_upload(handle, sec, chunk.ctypes.data, chunk.size, off),
                           "h2b_upload")
        # serialises the host-side enqueue (graph cache, workspace growth); on the device the
        # library orders every call after the handle's previous one, whatever the stream
        self._lock = threading.Lock()
        self._perm_t = None

    # ------------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    @property
    def shape(self):
        return (self.n, self.n)

    def device_bytes(self):
        return int(_abi.lib().h2b_device_bytes(self._h))

    def close(self):
        self._finalizer()

    def perm_tensor(self):
        torch = _torch()
        if self._perm_t is None:
            self._perm_t = torch.from_numpy(self.perm).to(f"cuda:{self.device}")
        return self._perm_t

    # ---- device-side (permuted order) --------------------------------
    def matvec_perm(self, xp, out=None, stream=None):
        """y_perm = S x_perm on device; xp: (N,) or (N, q) complex128 CUDA tensor."""
        torch = _torch()
        if xp.dtype != torch.complex128 or not xp.is_cuda:
            raise ValueError("matvec_perm expects a complex128 CUDA tensor")
        if xp.shape[0] != self.n or xp.dim() not in (1, 2):
            raise ValueError(f"expected ({self.n},) or ({self.n}, q) input")
        xp = xp.contiguous()
        q = 1 if xp.dim() == 1 else int(xp.shape[1])
        if out is None:
            out = torch.empty_like(xp)
        with self._lock:
            _abi.check(_abi.lib().h2b_matvec_perm(self._h, C.c_void_p(xp.data_ptr()),
                                                  C.c_void_p(out.data_ptr()), q,
                                                  _stream_handle(stream)), "h2b_matvec_perm")
        return out

    def gather(self, x, out=None, stream=None):
        """out = x[perm] on device (arith.py:113)."""
        torch = _torch()
        x = x.contiguous()
        q = 1 if x.dim() == 1 else int(x.shape[1])
        out = torch.empty_like(x) if out is None else out
        _abi.check(_abi.lib().h2b_gather_perm(self._h, C.c_void_p(x.data_ptr()),
                                              C.c_void_p(out.data_ptr()), q,
                                              _stream_handle(stream)), "h2b_gather_perm")
        return out

    def scatter(self, yp, out=None, stream=None):
        """out[perm] = yp on device (arith.py:115-116)."""
        torch = _torch()
        yp = yp.contiguous()
        q = 1 if yp.dim() == 1 else int(yp.shape[1])
        out = torch.empty_like(yp) if out is None else out
        _abi.check(_abi.lib().h2b_scatter_perm(self._h, C.c_void_p(yp.data_ptr()),
                                               C.c_void_p(out.data_ptr()), q,
                                               _stream_handle(stream)), "h2b_scatter_perm")
        return out

    # ---- host-side drop-in (original order, numpy) --------------------
    def matvec(self, x):
        x = np.asarray(x, dtype=np.complex128)
        if x.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}")
        return self._host_apply(x, 1)

    def matmat(self, X):
        X = np.asarray(X, dtype=np.complex128)
        if X.ndim != 2 or X.shape[0] != self.n:
            raise ValueError(f"expected ({self.n}, q) block")
        return self._host_apply(X, X.shape[1])

    def _host_apply(self, x, q):
        if q == 0:
            return np.empty_like(x)
        xc = np.ascontiguousarray(x)
        y = np.empty_like(xc)
        with self._lock:
            _abi.check(_abi.lib().h2b_matvec_host(self._h, xc.ctypes.data, y.ctypes.data, int(q)),
                       "h2b_matvec_host")
        return y

    __call__ = matvec


# ----------------------------------------------------------------------
# reference-shaped drop-ins
# ----------------------------------------------------------------------
_cache: dict = {}
_cache_lock = threading.Lock()


def as_operator(h2, device=0) -> H2Operator:
    """H2Operator for a reference H2Matrix / PackedH2 (packed once, cached by identity)."""
    if isinstance(h2, H2Operator):
        return h2
    key = (id(h2), int(device))
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0]() is h2:
            return hit[1]
        op = H2Operator(h2, device=device)
        try:
            ref = weakref.ref(h2, lambda _r, k=key: _cache.pop(k, None))
        except TypeError:  # not weak-referenceable: keep it alive with the operator
            ref = (lambda o=h2: o)
        _cache[key] = (ref, op)
        return op


def matvec(h2, x):
    """y = S x through the nested representation (drop-in for arith.matvec, arith.py:108-117)."""
    op = as_operator(h2)
    x = np.asarray(x, dtype=np.complex128)
    if x.shape != (op.n,):
        raise ValueError(f"expected vector of length {op.n}")
    return op.matvec(x)


def matmat_apply(h2, rhs_block, col_block=256):
    """Apply to an (n, q) block (drop-in for arith.matmat_apply, arith.py:120-130).

    The device applies all q columns at once; ``col_block`` only bounds the
    per-call column count (and thereby the workspace), as in the reference
    where chunking is invisible in the result.
    """
    op = as_operator(h2)
    rhs_block = np.asarray(rhs_block, dtype=np.complex128)
    if rhs_block.ndim != 2 or rhs_block.shape[0] != op.n:
        raise ValueError(f"expected ({op.n}, q) block")
    if col_block < 1:
        raise ValueError("col_block must be >= 1")
    out = np.empty_like(rhs_block)
    for j0 in range(0, rhs_block.shape[1], col_block):
        out[:, j0:j0 + col_block] = op.matmat(rhs_block[:, j0:j0 + col_block])
    return out
