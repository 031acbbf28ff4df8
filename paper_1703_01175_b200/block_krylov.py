"""Block GMRES(m) for q simultaneous right-hand sides, on device.

New component: the reference has no GMRES (SURVEY.md §0 finding 1; its only
solver is BiCGStab, arith.py:605-689), and BASELINE config 5 asks for a
block-GMRES over 64 plane-wave right-hand sides.  This follows the CPU
restatement ``oracle/krylov_oracle.py::block_gmres_solve`` step for step
(x0 = 0, block Arnoldi with block CGS2, QR of every new block, restart after
m blocks, converged when every column's TRUE relative residual is <= tol at
the end of a cycle; ``iterations`` counts block Arnoldi steps and the
history holds the max over columns of the least-squares residual relative to
||b_j||) so iteration counts agree with it.

Work split:
* the operator application is the H² matvec with q columns — libh2b's grouped
  complex GEMM on the FP64 tensor pipe (h2b_mrhs.cu), in the permuted space;
* the block Gram-Schmidt products V^H W, W - V H (tall-skinny complex GEMMs)
  and the QR of each new (N x q) block are plain dense library calls
  (cuBLAS ZGEMM / cuSOLVER via torch on the same stream);
* the small block-Hessenberg least-squares problem is solved incrementally:
  each new block column is rotated by the stored 2q x 2q unitary factors of
  the previous steps and the new ones come from a QR of its 2q x q bottom —
  the least-squares residual is then the norm of the rotated right-hand side's
  last q rows (mathematically the oracle's per-step lstsq residual).
"""

from __future__ import annotations

import time

import numpy as np

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
    dev = torch.device(f"cuda:{op.device}")
    n, q = B_h.shape
    bn_h = np.linalg.norm(B_h, axis=0)
    if np.all(bn_h == 0):
        return np.zeros_like(B_h), SolveReport(0, [], True, time.perf_counter() - t0)
    bn = torch.from_numpy(np.where(bn_h == 0, 1.0, bn_h)).to(dev)
    B = op.gather(torch.from_numpy(np.ascontiguousarray(B_h)).to(dev))
    m = int(restart)
    X = torch.zeros_like(B)
    Vbuf = torch.empty((n, (m + 1) * q), dtype=torch.complex128, device=dev)
    W = torch.empty_like(B)
    R = B.clone()
    it = 0
    history = []
    converged = False
    while it < max_iter:
        Q0, R0 = torch.linalg.qr(R)
        Vbuf[:, :q] = Q0
        E = torch.zeros(((m + 1) * q, q), dtype=torch.complex128, device=dev)
        E[:q] = R0
        U = torch.zeros((m * q, m * q), dtype=torch.complex128, device=dev)  # rotated H (upper)
        G = []
        j_done = 0
        for j in range(m):
            op.matvec_perm(Vbuf[:, j * q:(j + 1) * q].contiguous(), out=W)
            it += 1
            Vb = Vbuf[:, :(j + 1) * q]
            Hc = Vb.mH @ W
            W -= Vb @ Hc
            Hc2 = Vb.mH @ W
            W -= Vb @ Hc2
            Hc += Hc2
            Qj, Rj = torch.linalg.qr(W)
            Vbuf[:, (j + 1) * q:(j + 2) * q] = Qj
            h = torch.cat([Hc, Rj], dim=0)  # ((j+2)q, q) block column of H
            for i, Gi in enumerate(G):
                h[i * q:(i + 2) * q] = Gi.mH @ h[i * q:(i + 2) * q]
            Gj, Rt = torch.linalg.qr(h[j * q:(j + 2) * q], mode="complete")
            G.append(Gj)
            h[j * q:(j + 2) * q] = Rt
            U[:(j + 1) * q, j * q:(j + 1) * q] = h[:(j + 1) * q]
            E[j * q:(j + 2) * q] = Gj.mH @ E[j * q:(j + 2) * q]
            j_done = j + 1
            res = torch.linalg.vector_norm(E[(j + 1) * q:(j + 2) * q], dim=0) / bn
            rmax = float(res.max())
            history.append(rmax)
            if rmax <= tol or it >= max_iter:
                break
        k = j_done * q
        Y = torch.linalg.solve_triangular(U[:k, :k], E[:k], upper=True)
        X += Vbuf[:, :k] @ Y
        op.matvec_perm(X, out=W)
        R = B - W
        tr = torch.linalg.vector_norm(R, dim=0) / bn
        if float(tr.max()) <= tol:
            converged = True
            break
    Xh = op.scatter(X).cpu().numpy()
    return Xh, SolveReport(it, history, converged, time.perf_counter() - t0)
