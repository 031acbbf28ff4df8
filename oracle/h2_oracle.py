"""CPU oracle for the H² matvec hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or
as the timed reference CPU implementation.  The product path
(``paper_1703_01175_b200``) never routes through it.

This is a restatement, on the level-packed arrays of
``paper_1703_01175_b200.pack.PackedH2``, of the reference algorithm

* ``_apply_perm``  /root/reference/pkg/src/h2vie/arith.py:52-105
* ``matvec``       /root/reference/pkg/src/h2vie/arith.py:108-117
* ``matmat_apply`` /root/reference/pkg/src/h2vie/arith.py:120-130

with the reference's loop structure kept (one numpy ``@`` per block, Python
loops over levels, clusters and blocks), so that timing it measures what the
reference's CPU path costs.  A second, batched restatement
(`matvec_perm_packed`) groups equal-shape blocks into einsums; it exists to
cross-check the first by a different summation order.

Pinning: ``tests/test_oracle.py`` checks both against the golden vectors in
``tests/golden/`` which were produced by the reference itself
(``tools/make_golden.py`` imports ``h2vie`` from /root/reference and stores
``arith.matvec`` / ``arith.matmat_apply`` outputs).  Parity pinned.
"""

from __future__ import annotations

import numpy as np


def _apply_perm_loop(pk, xp):
    """Restates arith.py:52-104 on a PackedH2: xp is (N, q) in permuted order."""
    q = xp.shape[1]
    P = pk.num_clusters
    fwd = [None] * P
    # (1) forward transform, deepest level first (arith.py:58-71)
    for lvl in range(pk.depth - 1, -1, -1):
        for p in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            k = int(pk.c_rank[p])
            if k == 0:                                   # arith.py:62-65
                fwd[p] = np.zeros((0, q), dtype=np.complex128)
                continue
            if pk.c_child_lo[p] < 0:                     # leaf: V^T x (arith.py:66-67)
                n = int(pk.c_size[p])
                v = pk.vbuf[pk.c_v_off[p]:pk.c_v_off[p] + n * k].reshape(n, k)
                s0 = int(pk.c_start[p])
                fwd[p] = v.T @ xp[s0:s0 + n]
            else:                                        # T_lo^T x_lo + T_hi^T x_hi (:68-71)
                lo, hi = int(pk.c_child_lo[p]), int(pk.c_child_hi[p])
                klo, khi = int(pk.c_rank[lo]), int(pk.c_rank[hi])
                o = int(pk.c_t_off[p])
                t_lo = pk.tbuf[o:o + klo * k].reshape(klo, k)
                t_hi = pk.tbuf[o + klo * k:o + (klo + khi) * k].reshape(khi, k)
                fwd[p] = t_lo.T @ fwd[lo] + t_hi.T @ fwd[hi]
    # (2) coupling y^t += S^{t,s} x^s in sorted (t,s) order (arith.py:72-81)
    acc = [None] * P
    for t in range(P):
        kt = int(pk.c_rank[t])
        for b in range(pk.s_row_ptr[t], pk.s_row_ptr[t + 1]):
            s = int(pk.s_col[b])
            ks = int(pk.c_rank[s])
            if kt * ks == 0:                             # arith.py:75-76
                continue
            o = int(pk.s_off[b])
            smat = pk.sbuf[o:o + kt * ks].reshape(kt, ks)
            contrib = smat @ fwd[s]
            acc[t] = contrib if acc[t] is None else acc[t] + contrib
    # (3) backward transform, root level first (arith.py:82-99)
    yp = np.zeros((pk.n, q), dtype=np.complex128)
    for lvl in range(pk.depth):
        for p in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            ya = acc[p]
            if ya is None:
                continue
            k = int(pk.c_rank[p])
            if pk.c_child_lo[p] < 0:
                n = int(pk.c_size[p])
                v = pk.vbuf[pk.c_v_off[p]:pk.c_v_off[p] + n * k].reshape(n, k)
                s0 = int(pk.c_start[p])
                yp[s0:s0 + n] += v @ ya
            else:
                lo, hi = int(pk.c_child_lo[p]), int(pk.c_child_hi[p])
                klo, khi = int(pk.c_rank[lo]), int(pk.c_rank[hi])
                o = int(pk.c_t_off[p])
                t_lo = pk.tbuf[o:o + klo * k].reshape(klo, k)
                t_hi = pk.tbuf[o + klo * k:o + (klo + khi) * k].reshape(khi, k)
                for child, tr in ((lo, t_lo), (hi, t_hi)):
                    acc[child] = tr @ ya if acc[child] is None else acc[child] + tr @ ya
    # (4) dense inadmissible leaves (arith.py:100-104)
    for t in range(P):
        nt, t0 = int(pk.c_size[t]), int(pk.c_start[t])
        for b in range(pk.d_row_ptr[t], pk.d_row_ptr[t + 1]):
            s = int(pk.d_col[b])
            ns, s0 = int(pk.c_size[s]), int(pk.c_start[s])
            o = int(pk.d_off[b])
            d = pk.dbuf[o:o + nt * ns].reshape(nt, ns)
            yp[t0:t0 + nt] += d @ xp[s0:s0 + ns]
    return yp


def matvec_perm(pk, xp):
    """y_perm = S x_perm for a 1-D or (N, q) permuted-order input."""
    xp = np.asarray(xp, dtype=np.complex128)
    if xp.ndim == 1:
        return _apply_perm_loop(pk, xp[:, None])[:, 0]
    return _apply_perm_loop(pk, xp)


def matvec(pk, x):
    """Restates arith.matvec (arith.py:108-117)."""
    x = np.asarray(x, dtype=np.complex128)
    if x.shape != (pk.n,):
        raise ValueError(f"expected vector of length {pk.n}")
    yp = _apply_perm_loop(pk, x[pk.perm][:, None])[:, 0]
    y = np.empty_like(yp)
    y[pk.perm] = yp
    return y


def matmat_apply(pk, rhs_block, col_block=256):
    """Restates arith.matmat_apply (arith.py:120-130)."""
    rhs_block = np.asarray(rhs_block, dtype=np.complex128)
    if rhs_block.ndim != 2 or rhs_block.shape[0] != pk.n:
        raise ValueError(f"expected ({pk.n}, q) block")
    out = np.empty_like(rhs_block)
    for j0 in range(0, rhs_block.shape[1], col_block):
        chunk = rhs_block[pk.perm, j0:j0 + col_block]
        out[pk.perm, j0:j0 + col_block] = _apply_perm_loop(pk, chunk)
    return out


# ----------------------------------------------------------------------
# batched restatement (different summation order; cross-check only)
# ----------------------------------------------------------------------

def matvec_perm_packed(pk, xp):
    """Same operator, blocks grouped by shape and applied with einsum.

    Exists only to cross-check `_apply_perm_loop` through an independent
    code path (SURVEY.md §0 finding 2 measured 3e-16 agreement).
    """
    xp = np.asarray(xp, dtype=np.complex128)
    squeeze = xp.ndim == 1
    if squeeze:
        xp = xp[:, None]
    q = xp.shape[1]
    P = pk.num_clusters
    K = pk.total_rank
    xh = np.zeros((K, q), dtype=np.complex128)
    off = pk.c_xhat_off
    for lvl in range(pk.depth - 1, -1, -1):
        for p in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            k = int(pk.c_rank[p])
            if k == 0:
                continue
            if pk.c_child_lo[p] < 0:
                n, s0 = int(pk.c_size[p]), int(pk.c_start[p])
                v = pk.vbuf[pk.c_v_off[p]:pk.c_v_off[p] + n * k].reshape(n, k)
                xh[off[p]:off[p] + k] = np.einsum("ij,iq->jq", v, xp[s0:s0 + n])
            else:
                lo, hi = int(pk.c_child_lo[p]), int(pk.c_child_hi[p])
                klo, khi = int(pk.c_rank[lo]), int(pk.c_rank[hi])
                o = int(pk.c_t_off[p])
                t = pk.tbuf[o:o + (klo + khi) * k].reshape(klo + khi, k)
                src = np.concatenate([xh[off[lo]:off[lo] + klo], xh[off[hi]:off[hi] + khi]])
                xh[off[p]:off[p] + k] = np.einsum("ij,iq->jq", t, src)
    yh = np.zeros((K, q), dtype=np.complex128)
    rows = np.repeat(np.arange(P), np.diff(pk.s_row_ptr))
    for b in range(pk.n_coupling):
        t, s = rows[b], int(pk.s_col[b])
        kt, ks = int(pk.c_rank[t]), int(pk.c_rank[s])
        if kt * ks == 0:
            continue
        o = int(pk.s_off[b])
        yh[off[t]:off[t] + kt] += pk.sbuf[o:o + kt * ks].reshape(kt, ks) @ xh[off[s]:off[s] + ks]
    yp = np.zeros((pk.n, q), dtype=np.complex128)
    for lvl in range(pk.depth):
        for p in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            k = int(pk.c_rank[p])
            if k == 0:
                continue
            if pk.c_child_lo[p] < 0:
                n, s0 = int(pk.c_size[p]), int(pk.c_start[p])
                v = pk.vbuf[pk.c_v_off[p]:pk.c_v_off[p] + n * k].reshape(n, k)
                yp[s0:s0 + n] += np.einsum("ij,jq->iq", v, yh[off[p]:off[p] + k])
            else:
                lo, hi = int(pk.c_child_lo[p]), int(pk.c_child_hi[p])
                klo, khi = int(pk.c_rank[lo]), int(pk.c_rank[hi])
                o = int(pk.c_t_off[p])
                t = pk.tbuf[o:o + (klo + khi) * k].reshape(klo + khi, k)
                down = t @ yh[off[p]:off[p] + k]
                yh[off[lo]:off[lo] + klo] += down[:klo]
                yh[off[hi]:off[hi] + khi] += down[klo:]
    drows = np.repeat(np.arange(P), np.diff(pk.d_row_ptr))
    for b in range(pk.n_near):
        t, s = drows[b], int(pk.d_col[b])
        nt, ns = int(pk.c_size[t]), int(pk.c_size[s])
        t0, s0 = int(pk.c_start[t]), int(pk.c_start[s])
        o = int(pk.d_off[b])
        yp[t0:t0 + nt] += pk.dbuf[o:o + nt * ns].reshape(nt, ns) @ xp[s0:s0 + ns]
    return yp[:, 0] if squeeze else yp
