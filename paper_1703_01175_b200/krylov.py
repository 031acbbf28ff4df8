"""Krylov solvers on device, behind the reference's solver surface.

* `bicgstab_solve(apply, rhs, tol=1e-3, max_iter=200, seed=0, shadow=None)`
  — same signature, argument checks, breakdown-restart rule and
  `SolveReport` as ``h2vie.arith.bicgstab_solve`` (arith.py:605-689).
* `gmres_solve(apply, rhs, tol=1e-6, restart=30, max_iter=1000)` — new
  (the reference has no GMRES); restarted GMRES(m), CGS2, x0 = 0.

``apply`` is either the operator — an `H2Operator`, a reference ``H2Matrix``
or a `PackedH2` (wrapped once) — or any callable ``v -> A v`` on numpy
vectors, which is how the reference harness calls its solver
(``lambda v: arith.matvec(h2, v)``, bench.py:253-256,333-337).

* Operator: the whole iteration runs on the GPU in the cluster-permuted
  space (a permutation preserves inner products, so the iterates are those
  of the original ordering); only the RHS and the solution cross PCIe.
* Callable: the solver cannot see inside a host closure, so the recurrence
  is driven from the host on numpy vectors and every operator application is
  the caller's own call — with ``lambda v: matvec(h2, v)`` that is this
  package's GPU matvec (h2b_matvec_host).  Same recurrence, tests and
  reports as the device loop; this is the reference's own calling convention,
  not a CPU fallback (nothing here computes a matvec).
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
    """The device operator behind ``apply``, or None for an opaque callable."""
    if isinstance(apply, H2Operator):
        return apply
    if isinstance(apply, PackedH2) or (hasattr(apply, "tree") and hasattr(apply, "coupling")):
        return as_operator(apply)
    owner = getattr(apply, "__self__", None)  # a bound H2Operator.matvec
    if isinstance(owner, H2Operator) and getattr(apply, "__func__", None) is H2Operator.matvec:
        return owner
    if callable(apply):
        return None
    raise TypeError("apply must be an H2Operator, an H2Matrix, a PackedH2 or a callable v -> A v")


def _checked_apply(apply, n):
    def f(v):
        y = np.asarray(apply(v), dtype=np.complex128)
        if y.shape != (n,):
            raise ValueError(f"apply returned shape {y.shape}, expected ({n},)")
        return y
    return f


def _gmres_host(apply, b, tol, restart, max_iter, t0):
    """GMRES(m), CGS2, x0 = 0, driven from the host around a caller-supplied ``apply``.

    The same recurrence as the device loop (h2b_krylov.cu: h2b_gmres / givens_update): two
    classical Gram-Schmidt passes, complex Givens rotations with a real cosine, stop on the
    rotated residual |g_{j+1}| / ||b|| <= tol (or at a cycle end), then the true residual.
    """
    n = b.size
    bnrm = float(np.linalg.norm(b))
    if bnrm == 0.0:
        return np.zeros(n, dtype=np.complex128), SolveReport(0, [], True, time.perf_counter() - t0)
    m = int(restart)
    x = np.zeros(n, dtype=np.complex128)
    r = b.copy()
    it, history, converged = 0, [], False
    while it < max_iter:
        beta = float(np.linalg.norm(r))
        V = np.zeros((m + 1, n), dtype=np.complex128)
        R = np.zeros((m, m), dtype=np.complex128)   # rotated Hessenberg (upper triangle)
        c_rot = np.zeros(m)
        s_rot = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        for j in range(m):
            w = apply(V[j])
            it += 1
            h = V[:j + 1].conj() @ w
            w = w - h @ V[:j + 1]
            h2 = V[:j + 1].conj() @ w
            w = w - h2 @ V[:j + 1]
            h = h + h2
            hn = float(np.linalg.norm(w))
            for i in range(j):
                hi, hi1 = h[i], h[i + 1]
                h[i] = c_rot[i] * hi + s_rot[i] * hi1
                h[i + 1] = -np.conj(s_rot[i]) * hi + c_rot[i] * hi1
            ahj = abs(h[j])
            if hn == 0.0:
                c, s, rr = 1.0, 0j, h[j]
            elif ahj == 0.0:
                c, s, rr = 0.0, 1 + 0j, complex(hn)
            else:
                t = np.hypot(ahj, hn)
                ph = h[j] / ahj
                c, s, rr = ahj / t, ph * hn / t, ph * t
            c_rot[j], s_rot[j] = c, s
            R[:j + 1, j] = h[:j + 1]
            R[j, j] = rr
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            res = abs(g[j + 1]) / bnrm
            history.append(float(res))
            j_done = j + 1
            if res <= tol or it >= max_iter or hn == 0.0:
                break
            V[j + 1] = w / hn
        y = np.zeros(j_done, dtype=np.complex128)
        for i in range(j_done - 1, -1, -1):
            y[i] = (g[i] - R[i, i + 1:j_done] @ y[i + 1:j_done]) / R[i, i]
        x = x + y @ V[:j_done]
        r = b - apply(x)
        if float(np.linalg.norm(r)) / bnrm <= tol:
            converged = True
            break
    return x, SolveReport(it, history, converged, time.perf_counter() - t0)


def _bicgstab_host(apply, b, tol, max_iter, seed, shadow, t0):
    """BiCGStab driven from the host around a caller-supplied ``apply``: the reference
    recurrence (arith.py:605-689) — rho-breakdown restart with the seeded perturbation
    (:639-653), the early ||s|| exit (:666-670), the same SolveReport."""
    n = b.size
    bnrm = np.linalg.norm(b)
    if bnrm == 0.0:
        return np.zeros(n, dtype=np.complex128), SolveReport(0, [], True, time.perf_counter() - t0)
    x = np.zeros(n, dtype=np.complex128)
    r = b.copy()
    rh = r.copy() if shadow is None else np.asarray(shadow, dtype=np.complex128).copy()
    rho = alpha = omega = 1.0 + 0j
    v = np.zeros(n, dtype=np.complex128)
    p = np.zeros(n, dtype=np.complex128)
    thr = np.finfo(np.float64).eps ** 2 * max(1.0, bnrm ** 2)
    history, converged, restarted, it = [], False, False, 0
    while it < max_iter:
        it += 1
        rho_new = np.vdot(rh, r)
        if abs(rho_new) < thr:
            if restarted:
                break
            rng = np.random.default_rng(seed)
            rh = r + bnrm * 1e-8 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
            rho = alpha = omega = 1.0 + 0j
            v[:] = 0
            p[:] = 0
            restarted = True
            rho_new = np.vdot(rh, r)
            if abs(rho_new) < thr:
                break
        if it == 1 or not p.any():
            p = r.copy()
        else:
            beta = (rho_new / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
        v = apply(p)
        denom = np.vdot(rh, v)
        if denom == 0:
            break
        alpha = rho_new / denom
        s = r - alpha * v
        s_rel = np.linalg.norm(s) / bnrm
        if s_rel <= tol:
            x += alpha * p
            history.append(float(s_rel))
            converged = True
            break
        t = apply(s)
        tt = np.vdot(t, t)
        if tt == 0:
            break
        omega = np.vdot(t, s) / tt
        if omega == 0:
            break
        x += alpha * p + omega * s
        r = s - omega * t
        rho = rho_new
        rel = float(np.linalg.norm(r) / bnrm)
        history.append(rel)
        if rel <= tol:
            converged = True
            break
        if not np.isfinite(rel):
            break
    return x, SolveReport(it, history, converged, time.perf_counter() - t0)


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
    t0 = time.perf_counter()
    if op is None:
        if b.ndim != 1:
            raise ValueError("rhs must be a vector")
        return _gmres_host(_checked_apply(apply, b.size), b, tol, restart, max_iter, t0)
    if b.shape != (op.n,):
        raise ValueError(f"expected vector of length {op.n}")
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
    t0 = time.perf_counter()
    if op is None:
        if b.ndim != 1:
            raise ValueError("rhs must be a vector")
        return _bicgstab_host(_checked_apply(apply, b.size), b, tol, max_iter, seed, shadow, t0)
    if b.shape != (op.n,):
        raise ValueError(f"expected vector of length {op.n}")
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
