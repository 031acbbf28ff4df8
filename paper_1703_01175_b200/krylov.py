"""Krylov solvers on device, behind the reference's solver surface.

* `bicgstab_solve(apply, rhs, tol=1e-3, max_iter=200, seed=0, shadow=None)`
  — same signature, argument checks, breakdown-restart rule and
  `SolveReport` as ``h2vie.arith.bicgstab_solve`` (arith.py:605-689).
* `gmres_solve(apply, rhs, tol=1e-6, restart=30, max_iter=1000)` — new
  (the reference has no GMRES); restarted GMRES(m), CGS2, x0 = 0.

``apply`` is the operator: an `H2Operator`, a reference ``H2Matrix`` or a
`PackedH2` (wrapped once), i.e. what the reference harness passes as
``lambda v: arith.matvec(h2, v)`` (bench.py:253-256,333-337).  The whole
iteration runs on the GPU in the cluster-permuted space (a permutation
preserves inner products, so the iterates are those of the original
ordering); only the RHS and the solution cross PCIe.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _abi
from .h2op import H2Operator, as_operator, _stream_handle
from .pack import PackedH2


@dataclass
class SolveReport:
    """Same fields as h2vie.arith.SolveReport (arith.py:39-44)."""

    iterations: int
    residual_history: list
    converged: bool
    wall_time: float


def _operator_of(apply):
    if isinstance(apply, H2Operator):
        return apply
    if isinstance(apply, PackedH2) or (hasattr(apply, "tree") and hasattr(apply, "coupling")):
        return as_operator(apply)
    raise TypeError("apply must be an H2Operator, an H2Matrix or a PackedH2: the GPU solver "
                    "keeps the whole iteration on device and cannot call a host closure")


def _to_device_perm(op, vec):
    torch = __import__("torch")
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.complex128)).to(f"cuda:{op.device}")
    return op.gather(t)


def gmres_solve(apply, rhs, tol=1e-6, restart=30, max_iter=1000):
    """Restarted GMRES(restart) to ||r||/||b|| <= tol; returns (x, SolveReport)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be >= 1")
    op = _operator_of(apply)
    b = np.asarray(rhs, dtype=np.complex128)
    if b.shape != (op.n,):
        raise ValueError(f"expected vector of length {op.n}")
    t0 = time.perf_counter()
    torch = __import__("torch")
    bp = _to_device_perm(op, b)
    xp = torch.empty_like(bp)
    hist = np.zeros(max_iter, dtype=np.float64)
    rep = _abi.Report()
    with op._lock:
        _abi.check(_abi.lib().h2b_gmres(op.handle, C.c_void_p(bp.data_ptr()),
                                        C.c_void_p(xp.data_ptr()), int(restart), float(tol),
                                        int(max_iter), hist.ctypes.data_as(C.POINTER(C.c_double)),
                                        C.byref(rep), _stream_handle(None)), "h2b_gmres")
    x = op.scatter(xp).cpu().numpy()
    return x, SolveReport(int(rep.iterations), hist[:rep.n_history].tolist(), bool(rep.converged),
                          time.perf_counter() - t0)


def bicgstab_solve(apply, rhs, tol=1e-3, max_iter=200, seed=0, shadow=None):
    """Unpreconditioned BiCGStab (arith.py:605-689) with the loop on device."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    op = _operator_of(apply)
    b = np.asarray(rhs, dtype=np.complex128)
    if b.shape != (op.n,):
        raise ValueError(f"expected vector of length {op.n}")
    t0 = time.perf_counter()
    torch = __import__("torch")
    n = op.n
    bnrm = np.linalg.norm(b)
    bp = _to_device_perm(op, b)
    sp = _to_device_perm(op, shadow) if shadow is not None else None
    # the reference draws its restart perturbation from default_rng(seed) (arith.py:645-648);
    # the identical draw is made here and handed to the device loop (permuted, pre-scaled)
    rng = np.random.default_rng(seed)
    noise = bnrm * 1e-8 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    npn = _to_device_perm(op, noise)
    xp = torch.empty_like(bp)
    hist = np.zeros(max_iter, dtype=np.float64)
    rep = _abi.Report()
    with op._lock:
        _abi.check(_abi.lib().h2b_bicgstab(
            op.handle, C.c_void_p(bp.data_ptr()), C.c_void_p(xp.data_ptr()), float(tol),
            int(max_iter), C.c_void_p(sp.data_ptr()) if sp is not None else None,
            C.c_void_p(npn.data_ptr()), hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep),
            _stream_handle(None)), "h2b_bicgstab")
    x = op.scatter(xp).cpu().numpy()
    return x, SolveReport(int(rep.iterations), hist[:rep.n_history].tolist(), bool(rep.converged),
                          time.perf_counter() - t0)
