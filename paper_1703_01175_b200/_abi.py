"""ctypes binding of the C ABI in include/h2b.h (libh2b.so, built in-tree).

There is deliberately no fallback: if the library is missing or no
compute-capability-10 device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libh2b.so")

H2B_OK, H2B_EINVAL, H2B_ECUDA, H2B_ENOMEM, H2B_ESTATE, H2B_ENODEV = 0, -1, -2, -3, -4, -5
SEC_V, SEC_T, SEC_S, SEC_D = 0, 1, 2, 3

EXPORTED = (
    "h2b_version", "h2b_last_error", "h2b_device_ok", "h2b_create", "h2b_upload",
    "h2b_destroy", "h2b_device_bytes", "h2b_matvec_perm", "h2b_matvec_host",
    "h2b_gather_perm", "h2b_scatter_perm", "h2b_gmres", "h2b_bicgstab",
    "h2b_zdotc_multi", "h2b_zgemv_sub", "h2b_zaxpby", "h2b_matvec_phase",
    "h2b_prepare_handle", "h2b_set_option", "h2b_query", "h2b_get_trace",
    "h2b_plan_create", "h2b_plan_upload", "h2b_plan_set_phase", "h2b_plan_run",
    "h2b_plan_destroy", "h2b_plan_device_bytes", "h2b_assemble_near", "h2b_plan_set_peers",
    "h2b_plan_bcast_rows", "h2b_ipc_get_handle", "h2b_ipc_open", "h2b_ipc_close",
    "h2b_plan_set_peer_offset", "h2b_device_alloc", "h2b_device_free", "h2b_plan_set_gather",
    "h2b_plan_set_near_fast", "h2b_plan_set_couple_fast", "h2b_fill_synthetic_raw",
    "h2b_plan_fill_synthetic", "h2b_plan_fill_near", "h2b_tree_trace", "h2b_near_trace", "h2b_gmres_state_elems", "h2b_gmres_givens", "h2b_zscale_dev", "h2b_block_gmres", "h2b_stream_read", "h2b_spin_ns", "h2b_stamp_ns", "h2b_builder_create", "h2b_builder_ranks", "h2b_builder_fetch", "h2b_builder_destroy", "h2b_stage1_run", "h2b_stage1_fetch", "h2b_stage1_destroy", "h2b_stage1_device_ptrs", "h2b_exact_rows",
)
OPT_GRAPHS, OPT_MEGA, OPT_TRACE, OPT_DEBUG, OPT_MRHS, OPT_TREE = 1, 2, 3, 4, 5, 6
Q_LAUNCHES_Q1, Q_SPAN_MODE, Q_SPLIT_LEVEL, Q_TOP_STAGED, Q_DEVICE_BYTES = 1, 2, 3, 4, 5
Q_MEGA, Q_MEGA_TASKS, Q_MEGA_GRID, Q_MEGA_TIERS, Q_DEVICE_ERROR = 6, 7, 8, 9, 10
Q_NEAR_TASKS, Q_NEAR_STAGES, Q_NEAR_SMEM, Q_MEGA_SMEM, Q_NEAR_VARIANT = 11, 12, 13, 14, 15
Q_MRHS_LAUNCHES, Q_TREE = 16, 17

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class Layout(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("depth", C.c_int32), ("num_clusters", C.c_int32),
        ("level_ptr", _i32p), ("c_start", _i32p), ("c_size", _i32p), ("c_rank", _i32p),
        ("c_child_lo", _i32p), ("c_child_hi", _i32p), ("c_parent", _i32p),
        ("c_xhat_off", _i64p), ("c_v_off", _i64p), ("c_t_off", _i64p),
        ("n_coupling", C.c_int64), ("s_row_ptr", _i64p), ("s_col", _i32p), ("s_off", _i64p),
        ("n_near", C.c_int64), ("d_row_ptr", _i64p), ("d_col", _i32p), ("d_off", _i64p),
        ("perm", _i64p),
        ("v_elems", C.c_int64), ("t_elems", C.c_int64), ("s_elems", C.c_int64),
        ("d_elems", C.c_int64),
    ]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("n_history", C.c_int32),
                ("matvecs", C.c_int32), ("wall_time", C.c_double)]


# plan handles (h2b_plan_*): numpy record layouts of h2b_mm_item / h2b_mm_seg
import numpy as _np  # noqa: E402

MM_ITEM = _np.dtype([("c_row", "<i8"), ("m", "<i4"), ("seg0", "<i4"), ("nseg", "<i4"),
                     ("flags", "<i4"), ("pad", "<i8")])
MM_SEG = _np.dtype([("a_off", "<i8"), ("b_row", "<i8"), ("k", "<i4"), ("lda", "<i4"),
                    ("flags", "<i4"), ("pad", "<i4")])
NEAR_ITEM = _np.dtype([("y_off", "<i8"), ("b_first", "<i4"), ("nb", "<i4"), ("row0", "<i4"),
                      ("pad", "<i4")])
NEAR_BLK = _np.dtype([("d_off", "<i8"), ("x_off", "<i8")])
COUPLE_ITEM = _np.dtype([("panel", "<i8"), ("xcol", "<i8"), ("out", "<i8"), ("R", "<i4"), ("w", "<i4")])
B_X, B_XHAT, B_YHAT, B_Y = 0, 1, 2, 3
ITEM_ACC, ITEM_BCAST = 256, 512
PLAN_PHASE_NEAR_FAST = 6  # h2b.h H2B_PLAN_PHASE_NEAR_FAST


class H2BError(RuntimeError):
    """A non-OK status from libh2b; .code holds the H2B_* value."""

    def __init__(self, msg, code):
        super().__init__(msg)
        self.code = code


_lib = None


def lib():
    """Load libh2b.so once; raise if it is missing (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first; "
                          "the H2 hot path has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.h2b_version.restype = C.c_int
    L.h2b_last_error.restype = C.c_char_p
    L.h2b_device_ok.argtypes = [C.c_int]
    L.h2b_create.argtypes = [C.POINTER(Layout), C.c_int, C.POINTER(vp)]
    L.h2b_upload.argtypes = [vp, C.c_int, vp, C.c_size_t, C.c_size_t]
    L.h2b_destroy.argtypes = [vp]
    L.h2b_device_bytes.argtypes = [vp]
    L.h2b_device_bytes.restype = C.c_int64
    L.h2b_matvec_perm.argtypes = [vp, vp, vp, C.c_int, vp]
    L.h2b_matvec_host.argtypes = [vp, vp, vp, C.c_int]
    L.h2b_gather_perm.argtypes = [vp, vp, vp, C.c_int, vp]
    L.h2b_scatter_perm.argtypes = [vp, vp, vp, C.c_int, vp]
    L.h2b_gmres.argtypes = [vp, vp, vp, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double),
                            C.POINTER(Report), vp]
    L.h2b_bicgstab.argtypes = [vp, vp, vp, C.c_double, C.c_int, vp, vp, C.POINTER(C.c_double),
                               C.POINTER(Report), vp]
    L.h2b_zdotc_multi.argtypes = [vp, C.c_int64, C.c_int, vp, C.c_int64, vp, vp]
    L.h2b_zgemv_sub.argtypes = [vp, C.c_int64, C.c_int, vp, vp, C.c_int64, vp, vp]
    L.h2b_matvec_phase.argtypes = [vp, C.c_int, vp, vp, C.c_int, vp]
    L.h2b_prepare_handle.argtypes = [vp]
    L.h2b_set_option.argtypes = [vp, C.c_int, C.c_int]
    L.h2b_query.argtypes = [vp, C.c_int, C.POINTER(C.c_int64)]
    L.h2b_get_trace.argtypes = [vp, C.POINTER(C.c_int64), C.c_int64]
    L.h2b_zaxpby.argtypes = [C.c_int64, C.c_double, C.c_double, vp, C.c_double, C.c_double, vp, vp]
    L.h2b_gmres_state_elems.argtypes = [C.c_int]
    L.h2b_gmres_state_elems.restype = C.c_int64
    L.h2b_gmres_givens.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    L.h2b_zscale_dev.argtypes = [vp, C.c_int64, vp, vp]
    L.h2b_block_gmres.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_double, C.c_int, vp, vp, vp]
    L.h2b_stream_read.argtypes = [vp, C.c_size_t, vp, vp]
    L.h2b_spin_ns.argtypes = [C.c_uint64, vp]
    L.h2b_builder_create.argtypes = [C.c_int, C.c_int] + [vp] * 18 + [C.c_double, C.c_int, vp]
    L.h2b_builder_ranks.argtypes = [vp, vp]
    L.h2b_builder_fetch.argtypes = [vp, C.c_int, vp, vp]
    L.h2b_builder_destroy.argtypes = [vp]
    L.h2b_stage1_run.argtypes = [C.c_int] + [vp] * 3 + [C.c_int64] + [vp] * 4 + [C.c_double, C.c_double, C.c_double,
                                                                             C.c_int, C.c_int] + [vp] * 8
    L.h2b_stage1_fetch.argtypes = [vp, vp, vp, vp]
    L.h2b_stage1_destroy.argtypes = [vp]
    L.h2b_stage1_device_ptrs.argtypes = [vp, vp, vp, vp]
    L.h2b_exact_rows.argtypes = [vp, C.c_int, C.c_int64, vp, vp, C.c_double, C.c_double, C.c_double, C.c_double,
                                 vp, vp, C.c_int]
    L.h2b_assemble_near.argtypes = [vp, vp, vp, C.c_double, C.c_double, C.c_double, C.c_double]
    L.h2b_plan_create.argtypes = [C.c_int, C.c_int, _i64p, C.POINTER(vp)]
    L.h2b_plan_upload.argtypes = [vp, C.c_int, vp, C.c_size_t, C.c_size_t]
    L.h2b_plan_set_phase.argtypes = [vp, C.c_int, C.c_int, _i64p, vp, C.c_int64, vp, C.c_int64]
    L.h2b_plan_run.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp]
    L.h2b_plan_destroy.argtypes = [vp]
    L.h2b_plan_set_peers.argtypes = [vp, C.POINTER(vp), C.c_int]
    L.h2b_plan_bcast_rows.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int, vp]
    L.h2b_ipc_get_handle.argtypes = [vp, vp]
    L.h2b_ipc_open.argtypes = [vp, C.POINTER(vp)]
    L.h2b_ipc_close.argtypes = [vp]
    L.h2b_plan_set_peer_offset.argtypes = [vp, C.c_int64]
    L.h2b_plan_set_gather.argtypes = [vp, C.POINTER(C.c_int32), C.c_int64]
    L.h2b_fill_synthetic_raw.argtypes = [vp, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_double]
    L.h2b_plan_fill_synthetic.argtypes = [vp, C.c_int, vp, C.c_int64, C.c_uint64, C.c_double]
    L.h2b_plan_fill_near.argtypes = [vp, C.c_int, vp, C.c_int64, vp, C.c_int64, vp, vp, C.c_double,
                                     C.c_double, C.c_double, C.c_double]
    L.h2b_plan_set_couple_fast.argtypes = [vp, vp, C.c_int64, C.POINTER(C.c_int32), C.c_int64]
    L.h2b_plan_set_near_fast.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, C.c_int, C.c_int]
    L.h2b_device_alloc.argtypes = [C.c_int, C.c_size_t, C.POINTER(vp)]
    L.h2b_device_free.argtypes = [vp]
    L.h2b_plan_device_bytes.argtypes = [vp]
    L.h2b_plan_device_bytes.restype = C.c_int64
    _lib = L
    return L


def check(rc, what=""):
    if rc != H2B_OK:
        msg = lib().h2b_last_error().decode(errors="replace")
        if rc == H2B_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise H2BError(f"{what}: {msg} (status {rc})", rc)
    return rc


def exported_symbols():
    """Names from include/h2b.h that the loaded library actually exports."""
    L = lib()
    out = []
    for name in EXPORTED:
        try:
            getattr(L, name)
            out.append(name)
        except AttributeError:
            pass
    return out
