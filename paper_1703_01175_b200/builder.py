"""Stage II of the H² builder on the device (first step).

Given the block structure (cluster tree and partition, as packed tables) and the Stage-I grouped
factors of every cluster — A_c (n_c x r), B_c (its partners' rows x r) and M_c = B_c^T conj(B_c),
the output of the reference's ``build_all_cluster_ab`` (build.py:190-225) — the nested bases,
transfer matrices and coupling matrices are computed on the B200 (csrc/h2b_build.cu:
``h2b_builder_create``), restating ``build_bases`` / ``build_coupling`` (build.py:228-309) and
``trunc_eig_hermitian`` (linalg.py:207-231).  The result is a `PackedH2` ready for
`H2Operator`; the near-field payload is taken from the structure operator (or re-assembled
from the geometry on the device).

Eigenvectors are unique only up to phases (and rotations inside degenerate eigenspaces), so the
bases differ from the reference's by unitary factors; the operator itself agrees to the
compression tolerance.
"""

from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _abi
from .pack import PackedH2


def build_stage2(pk: PackedH2, stage1: dict, eps_acc: float, device: int = 0) -> PackedH2:
    """Nested bases / transfers / couplings of ``pk``'s block structure from Stage-I factors.

    ``stage1``: ``s1_rank`` (r per cluster, packed order), ``s1_a`` / ``s1_a_off``,
    ``s1_m`` / ``s1_m_off``, ``s1_b`` / ``s1_b_off`` (flattened row-major factors),
    ``s1_part_ptr`` / ``s1_partner`` / ``s1_prow`` (each cluster's partners, packed index, and
    the first row of the partner's block in B) — see tools/make_stage1.py.
    """
    L = _abi.lib()
    if not L.h2b_device_ok(int(device)):
        raise RuntimeError("no sm_100 (B200) CUDA device visible; the builder has no CPU fallback")
    P = pk.num_clusters

    def a(name, dtype):
        return np.ascontiguousarray(stage1[name], dtype=dtype)

    dev = stage1.get("s1_device")  # (A, B, M) device pointers of a device Stage I: no host round trip
    empty = np.zeros(1, np.complex128)
    keep = dict(
        level_ptr=np.ascontiguousarray(pk.level_ptr, np.int32), c_start=np.ascontiguousarray(pk.c_start, np.int32),
        c_size=np.ascontiguousarray(pk.c_size, np.int32), c_lo=np.ascontiguousarray(pk.c_child_lo, np.int32),
        c_hi=np.ascontiguousarray(pk.c_child_hi, np.int32), c_par=np.ascontiguousarray(pk.c_parent, np.int32),
        r=a("s1_rank", np.int32), a_off=a("s1_a_off", np.int64),
        A=empty if dev else a("s1_a", np.complex128),
        m_off=a("s1_m_off", np.int64), M=empty if dev else a("s1_m", np.complex128), b_off=a("s1_b_off", np.int64),
        B=empty if dev else a("s1_b", np.complex128), pp=a("s1_part_ptr", np.int64), partner=a("s1_partner", np.int32),
        prow=a("s1_prow", np.int64), s_row_ptr=np.ascontiguousarray(pk.s_row_ptr, np.int64),
        s_col=np.ascontiguousarray(pk.s_col, np.int32))
    p = {k: v.ctypes.data for k, v in keep.items()}
    if dev:
        p["A"], p["B"], p["M"] = dev
    h = C.c_void_p()
    _abi.check(L.h2b_builder_create(P, int(pk.depth), p["level_ptr"], p["c_start"], p["c_size"], p["c_lo"],
                                    p["c_hi"], p["c_par"], p["r"], p["a_off"], p["A"], p["m_off"], p["M"],
                                    p["b_off"], p["B"], p["pp"], p["partner"], p["prow"], p["s_row_ptr"],
                                    p["s_col"], float(eps_acc), int(device), C.byref(h)), "h2b_builder_create")
    try:
        k = np.zeros(P, np.int32)
        _abi.check(L.h2b_builder_ranks(h, k.ctypes.data), "h2b_builder_ranks")
        lo, hi = pk.c_child_lo, pk.c_child_hi
        c_v_off = np.full(P, -1, np.int64)
        c_t_off = np.full(P, -1, np.int64)
        voff = toff = 0
        for c in range(P):
            if lo[c] < 0:
                c_v_off[c] = voff
                voff += int(pk.c_size[c]) * int(k[c])
            else:
                c_t_off[c] = toff
                toff += (int(k[lo[c]]) + int(k[hi[c]])) * int(k[c])
        rows = np.repeat(np.arange(P), np.diff(pk.s_row_ptr))
        sz = k[rows].astype(np.int64) * k[pk.s_col].astype(np.int64)
        s_off = np.zeros(len(sz), np.int64)
        if len(sz):
            s_off[1:] = np.cumsum(sz)[:-1]
        vbuf = np.empty(voff, np.complex128)
        tbuf = np.empty(toff, np.complex128)
        sbuf = np.empty(int(sz.sum()), np.complex128)
        for what, buf in ((0, vbuf), (1, tbuf), (2, sbuf)):
            if buf.size:
                _abi.check(L.h2b_builder_fetch(h, what, keep["c_lo"].ctypes.data, buf.ctypes.data),
                           "h2b_builder_fetch")
    finally:
        L.h2b_builder_destroy(h)
    xoff = np.zeros(P + 1, np.int64)
    np.cumsum(k, out=xoff[1:])
    meta = {k: v for k, v in pk.meta.items() if k != "synthetic"}  # real payloads now
    meta.update(built_on_device=True, eps_acc=float(eps_acc))
    return dataclasses.replace(pk, c_rank=k.astype(pk.c_rank.dtype), c_xhat_off=xoff, c_v_off=c_v_off,
                               c_t_off=c_t_off, s_off=s_off, vbuf=vbuf, tbuf=tbuf, sbuf=sbuf, meta=meta)


def stage1_device(pk: PackedH2, centers, chi, k0: float, volume: float, eps_aca: float, max_rank: int = 200,
                  device: int = 0, keep_on_device: bool = False) -> dict:
    """Stage I on the device: the ACA factors of every cluster's grouped admissible block row
    (csrc/h2b_build.cu: ``h2b_stage1_run``, restating linalg.aca_factorize), as the dict
    `build_stage2` takes.  ``centers`` (N x 3) and ``chi`` (N) in the original point order."""
    L = _abi.lib()
    if not L.h2b_device_ok(int(device)):
        raise RuntimeError("no sm_100 (B200) CUDA device visible; the builder has no CPU fallback")
    P = pk.num_clusters
    nb = int(pk.s_row_ptr[-1])
    keep = dict(c_start=np.ascontiguousarray(pk.c_start, np.int32), c_size=np.ascontiguousarray(pk.c_size, np.int32),
                perm=np.ascontiguousarray(pk.perm, np.int64), s_row_ptr=np.ascontiguousarray(pk.s_row_ptr, np.int64),
                s_col=np.ascontiguousarray(pk.s_col, np.int32),
                centers=np.ascontiguousarray(centers, np.float64), chi=np.ascontiguousarray(chi, np.complex128),
                rank=np.zeros(P, np.int32), a_off=np.zeros(P + 1, np.int64), b_off=np.zeros(P + 1, np.int64),
                m_off=np.zeros(P + 1, np.int64), part_ptr=np.zeros(P + 1, np.int64),
                partner=np.zeros(max(nb, 1), np.int32), prow=np.zeros(max(nb, 1), np.int64))
    p = {k: v.ctypes.data for k, v in keep.items()}
    h = C.c_void_p()
    _abi.check(L.h2b_stage1_run(P, p["c_start"], p["c_size"], p["perm"], int(pk.n), p["s_row_ptr"], p["s_col"],
                                p["centers"], p["chi"], float(k0), float(volume), float(eps_aca), int(max_rank),
                                int(device), p["rank"], p["a_off"], p["b_off"], p["m_off"], p["part_ptr"],
                                p["partner"], p["prow"], C.byref(h)), "h2b_stage1_run")
    out = dict(s1_rank=keep["rank"], s1_a_off=keep["a_off"], s1_b_off=keep["b_off"], s1_m_off=keep["m_off"],
               s1_part_ptr=keep["part_ptr"], s1_partner=keep["partner"][:nb], s1_prow=keep["prow"][:nb])
    if keep_on_device:  # the caller releases the factors with h2b_stage1_destroy(out["s1_handle"])
        pa, pb, pm = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _abi.check(L.h2b_stage1_device_ptrs(h, C.byref(pa), C.byref(pb), C.byref(pm)), "h2b_stage1_device_ptrs")
        out.update(s1_device=(pa.value, pb.value, pm.value), s1_handle=h)
        return out
    try:
        A = np.empty(int(keep["a_off"][-1]), np.complex128)
        B = np.empty(int(keep["b_off"][-1]), np.complex128)
        M = np.empty(int(keep["m_off"][-1]), np.complex128)
        _abi.check(L.h2b_stage1_fetch(h, A.ctypes.data, B.ctypes.data, M.ctypes.data), "h2b_stage1_fetch")
    finally:
        L.h2b_stage1_destroy(h)
    out.update(s1_a=A, s1_b=B, s1_m=M)
    return out


def build_device(pk: PackedH2, centers, chi, k0: float, volume: float, eps_aca: float, eps_acc: float,
                 max_rank: int = 200, device: int = 0) -> PackedH2:
    """The far field of ``pk``'s block structure built on the device: Stage I (ACA) then Stage II
    (bases, transfers, couplings).  The near-field payload of ``pk`` is kept (or, when it is empty,
    sampled from the geometry on the device by `H2Operator`)."""
    s1 = stage1_device(pk, centers, chi, k0, volume, eps_aca, max_rank, device, keep_on_device=True)
    try:
        return build_stage2(pk, s1, eps_acc, device)
    finally:
        _abi.lib().h2b_stage1_destroy(s1["s1_handle"])


def exact_rows(rows, x, centers, chi, k0: float, volume: float, device: int = 0):
    """(S x)[rows] of the exact system matrix (kernel.py:190-210 entries incl. the self term,
    summed over all N columns on the device): the dense reference for sampled rows."""
    from .nearfield import self_term
    L = _abi.lib()
    rows = np.ascontiguousarray(rows, np.int64)
    x = np.ascontiguousarray(x, np.complex128)
    centers = np.ascontiguousarray(centers, np.float64)
    chi = np.ascontiguousarray(chi, np.complex128)
    diag = k0 ** 2 * self_term(volume, k0)
    out = np.empty(rows.size, np.complex128)
    _abi.check(L.h2b_exact_rows(rows.ctypes.data, int(rows.size), int(x.size), centers.ctypes.data, chi.ctypes.data,
                                float(k0), float(volume), float(diag.real), float(diag.imag), x.ctypes.data,
                                out.ctypes.data, int(device)), "h2b_exact_rows")
    return out
