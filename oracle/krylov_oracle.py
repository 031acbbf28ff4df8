"""CPU oracle for the Krylov loop around the matvec — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may use this module.

* `bicgstab_solve` restates the reference's own solver line by line
  (/root/reference/pkg/src/h2vie/arith.py:605-689, report type :39-44).
* `gmres_solve` is NEW: the reference has no GMRES (SURVEY.md §0 finding 1).
  It is a textbook restarted GMRES(m) with classical Gram-Schmidt applied
  twice (CGS2), x0 = 0, complex Givens rotations, stop when the rotated
  residual estimate |g_{j+1}|/||b|| <= tol and then confirm with the true
  residual; restart otherwise.  Its iteration count is cross-checked against
  `scipy.sparse.linalg.gmres(rtol=tol, atol=0, restart=m)` in
  ``tests/test_oracle.py`` (245 iterations on config 1 for
  MGS, CGS2 and scipy alike).  Parity of GMRES is therefore pinned to scipy,
  not to the reference, which has none.
* `block_gmres_solve`: block GMRES(m) for q right-hand sides (BASELINE
  config 5), a block-Arnoldi restatement; no external oracle exists.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np


@dataclass
class SolveReport:
    """Same fields as h2vie.arith.SolveReport (arith.py:39-44)."""

    iterations: int
    residual_history: list
    converged: bool
    wall_time: float


def bicgstab_solve(apply, rhs, tol=1e-3, max_iter=200, seed=0, shadow=None):
    """Restates arith.bicgstab_solve (arith.py:605-689)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    t_start = time.perf_counter()
    b = np.asarray(rhs, dtype=np.complex128)
    n = b.size
    bnrm = np.linalg.norm(b)
    if bnrm == 0.0:
        return np.zeros(n, dtype=np.complex128), SolveReport(0, [], True, time.perf_counter() - t_start)
    x = np.zeros(n, dtype=np.complex128)
    r = b.copy()
    r_hat = r.copy() if shadow is None else np.asarray(shadow, dtype=np.complex128).copy()
    rho = alpha = omega = 1.0 + 0j
    v = np.zeros(n, dtype=np.complex128)
    p = np.zeros(n, dtype=np.complex128)
    history = []
    converged = False
    restarted = False
    it = 0
    breakdown = np.finfo(np.float64).eps ** 2
    while it < max_iter:
        it += 1
        rho_new = np.vdot(r_hat, r)
        if abs(rho_new) < breakdown * max(1.0, bnrm ** 2):       # arith.py:639-653
            if restarted:
                break
            rng = np.random.default_rng(seed)
            r_hat = r + bnrm * 1e-8 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
            rho = alpha = omega = 1.0 + 0j
            v[:] = 0
            p[:] = 0
            restarted = True
            rho_new = np.vdot(r_hat, r)
            if abs(rho_new) < breakdown * max(1.0, bnrm ** 2):
                break
        if it == 1 or np.all(p == 0):
            p = r.copy()
        else:
            beta = (rho_new / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
        v = apply(p)
        denom = np.vdot(r_hat, v)
        if denom == 0:
            break
        alpha = rho_new / denom
        s = r - alpha * v
        s_nrm = np.linalg.norm(s)
        if s_nrm / bnrm <= tol:                                   # arith.py:666-670
            x += alpha * p
            history.append(float(s_nrm / bnrm))
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
    return x, SolveReport(it, history, converged, time.perf_counter() - t_start)


def givens(a, b):
    """Complex rotation (c real, s complex) with [c s; -conj(s) c] [a; b] = [r; 0], b real >= 0."""
    if b == 0.0:
        return 1.0, 0.0 + 0.0j, a
    if a == 0:
        return 0.0, 1.0 + 0.0j, complex(b)
    t = np.hypot(abs(a), b)
    ph = a / abs(a)
    return abs(a) / t, ph * b / t, ph * t


def gmres_solve(apply, rhs, tol=1e-6, restart=30, max_iter=1000):
    """Restarted GMRES(m), CGS2 Arnoldi, x0 = 0.  Returns (x, SolveReport)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must be in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be >= 1")
    t0 = time.perf_counter()
    b = np.asarray(rhs, dtype=np.complex128)
    n = b.size
    bnrm = float(np.linalg.norm(b))
    if bnrm == 0.0:
        return np.zeros(n, dtype=np.complex128), SolveReport(0, [], True, time.perf_counter() - t0)
    m = int(restart)
    x = np.zeros(n, dtype=np.complex128)
    r = b.copy()
    it = 0
    history = []
    converged = False
    while it < max_iter:
        beta = float(np.linalg.norm(r))
        V = np.zeros((m + 1, n), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        j_done = 0
        est_ok = False
        for j in range(m):
            w = apply(V[j])
            it += 1
            h = V[:j + 1].conj() @ w                 # CGS pass 1
            w = w - h @ V[:j + 1]
            h2 = V[:j + 1].conj() @ w                # CGS pass 2
            w = w - h2 @ V[:j + 1]
            h = h + h2
            hn = float(np.linalg.norm(w))
            for i in range(j):                       # previous rotations
                a, bb = h[i], h[i + 1]
                h[i] = cs[i] * a + sn[i] * bb
                h[i + 1] = -np.conj(sn[i]) * a + cs[i] * bb
            c, s, rr = givens(h[j], hn)
            cs[j], sn[j] = c, s
            H[:j + 1, j] = h
            H[j, j] = rr
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            res = abs(g[j + 1]) / bnrm
            history.append(float(res))
            j_done = j + 1
            if res <= tol:
                est_ok = True
                break
            if it >= max_iter or hn == 0.0:
                break
            V[j + 1] = w / hn
        y = np.zeros(j_done, dtype=np.complex128)   # back substitution
        for i in range(j_done - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:j_done]) / H[i, i]
        x = x + y @ V[:j_done]
        r = b - apply(x)
        true_res = float(np.linalg.norm(r)) / bnrm
        if est_ok and true_res <= tol:
            converged = True
            break
        if true_res <= tol:
            converged = True
            break
    return x, SolveReport(it, history, converged, time.perf_counter() - t0)


def block_gmres_solve(apply_block, rhs, tol=1e-6, restart=30, max_iter=1000):
    """Block GMRES(m) for (N, q) right-hand sides, x0 = 0.

    Block Arnoldi with block CGS2 + Householder-free QR (numpy.linalg.qr) of
    each new block; the small least-squares problem is solved with a dense
    QR per restart cycle.  Converged when every column's relative residual
    (true, recomputed at the end of a cycle) is <= tol; the per-iteration
    history holds the max over columns of the least-squares residual norm
    relative to ||b_j||.  `iterations` counts block Arnoldi steps.
    """
    t0 = time.perf_counter()
    B = np.asarray(rhs, dtype=np.complex128)
    if B.ndim != 2:
        raise ValueError("rhs must be (N, q)")
    n, q = B.shape
    bn = np.linalg.norm(B, axis=0)
    if np.all(bn == 0):
        return np.zeros_like(B), SolveReport(0, [], True, time.perf_counter() - t0)
    bn = np.where(bn == 0, 1.0, bn)
    X = np.zeros_like(B)
    R = B.copy()
    m = int(restart)
    it = 0
    history = []
    converged = False
    while it < max_iter:
        Q0, R0 = np.linalg.qr(R)
        V = [Q0]
        H = np.zeros(((m + 1) * q, m * q), dtype=np.complex128)
        E = np.zeros(((m + 1) * q, q), dtype=np.complex128)
        E[:q] = R0
        j_done = 0
        for j in range(m):
            W = apply_block(V[j])
            it += 1
            Vb = np.concatenate(V, axis=1)
            Hc = Vb.conj().T @ W
            W = W - Vb @ Hc
            Hc2 = Vb.conj().T @ W
            W = W - Vb @ Hc2
            Hc = Hc + Hc2
            Qj, Rj = np.linalg.qr(W)
            H[:(j + 1) * q, j * q:(j + 1) * q] = Hc
            H[(j + 1) * q:(j + 2) * q, j * q:(j + 1) * q] = Rj
            V.append(Qj)
            j_done = j + 1
            Hs = H[:(j + 2) * q, :(j + 1) * q]
            Y, *_ = np.linalg.lstsq(Hs, E[:(j + 2) * q], rcond=None)
            res = np.linalg.norm(E[:(j + 2) * q] - Hs @ Y, axis=0) / bn
            history.append(float(res.max()))
            if res.max() <= tol or it >= max_iter:
                break
        Hs = H[:(j_done + 1) * q, :j_done * q]
        Y, *_ = np.linalg.lstsq(Hs, E[:(j_done + 1) * q], rcond=None)
        X = X + np.concatenate(V[:j_done], axis=1) @ Y
        R = B - apply_block(X)
        tr = np.linalg.norm(R, axis=0) / bn
        if tr.max() <= tol:
            converged = True
            break
    return X, SolveReport(it, history, converged, time.perf_counter() - t0)
