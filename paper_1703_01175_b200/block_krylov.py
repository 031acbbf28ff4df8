"""Block GMRES(m) for q simultaneous right-hand sides, on device.

New component: the reference has no GMRES (SURVEY.md §0 finding 1; its only
solver is BiCGStab, arith.py:605-689), and BASELINE config 5 asks for a
block-GMRES over 64 plane-wave right-hand sides.  This follows the CPU
restatement ``oracle/krylov_oracle.py::block_gmres_solve`` step for step
(x0 = 0, block Arnoldi with block CGS2, a QR of every new block, restart after
m blocks, converged when every column's TRUE relative residual is <= tol at
the end of a cycle; ``iterations`` counts block Arnoldi steps and the history
holds the max over columns of the least-squares residual relative to ||b_j||)
so iteration counts agree with it.

The whole solve is ONE libh2b call (``h2b_block_gmres``, csrc/h2b_bkrylov.cu):
the q-column matvec on the FP64 tensor pipe, the tall-skinny block products
and CholQR2 of each block as libh2b kernels, and the small least-squares
problem orthonormalised incrementally on the device; the host reads each
step's residual from mapped pinned memory one step behind the GPU.  Right-hand
sides are processed in groups of at most 64 columns.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _abi
from .h2op import _stream_handle
from .krylov import SolveReport, _operator_of


def block_gmres_solve(apply_block, rhs, tol=1e-6, restart=30, max_iter=1000):
    """Block GMRES(restart) for an (N, q) right-hand side; returns (X, SolveReport)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be >= 1")
    op = _operator_of(apply_block)
    if op is None:
        raise TypeError("block_gmres_solve needs the operator (H2Operator / H2Matrix / PackedH2)")
    B_h = np.asarray(rhs, dtype=np.complex128)
    if B_h.ndim != 2 or B_h.shape[0] != op.n:
        raise ValueError(f"rhs must be ({op.n}, q)")
    import torch

    t0 = time.perf_counter()
    n, q = B_h.shape
    if q > 64:  # groups of 64 columns (independent block solves)
        Xs, reps = [], []
        for c0 in range(0, q, 64):
            X, r = block_gmres_solve(op, B_h[:, c0:c0 + 64], tol, restart, max_iter)
            Xs.append(X)
            reps.append(r)
        hist = [max(v) for v in zip(*[r.residual_history for r in reps])] if reps else []
        return np.concatenate(Xs, 1), SolveReport(max(r.iterations for r in reps), hist,
                                                  all(r.converged for r in reps), time.perf_counter() - t0)
    dev = torch.device(f"cuda:{op.device}")
    B = op.gather(torch.from_numpy(np.ascontiguousarray(B_h)).to(dev))
    X = torch.empty_like(B)
    hist = np.zeros(max_iter, dtype=np.float64)
    rep = _abi.Report()
    with op._lock:
        _abi.check(_abi.lib().h2b_block_gmres(op.handle, C.c_void_p(B.data_ptr()), C.c_void_p(X.data_ptr()),
                                              int(q), int(restart), float(tol), int(max_iter),
                                              hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep),
                                              _stream_handle(None)), "h2b_block_gmres")
    Xh = op.scatter(X).cpu().numpy()
    return Xh, SolveReport(int(rep.iterations), hist[:rep.n_history].tolist(), bool(rep.converged),
                           time.perf_counter() - t0)
