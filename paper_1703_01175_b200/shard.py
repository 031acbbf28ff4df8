"""Subtree partition of the H² operator across G ranks (one process per GPU).

SURVEY.md §8(e): for G = 2^p ranks, rank g owns the level-p cluster
``tree.levels[p][g]`` — a contiguous slice of the permuted index space
(clustering.py:87 splits at ``start + (n+1)//2``, so slices differ by at
most one point) — and everything below it: the leaf bases and transfers of
its subtree, the coupling rows S^{t,s} of its targets t, the near-field rows
D_{t,s} of its leaves.  Levels above p ("top") are tiny (the 3-D configs have
k = 0 there) and are computed redundantly by every rank.

One matvec on rank g (reference phases, arith.py:52-104):

1. ``UP_OWN``   x̂ of its own clusters from its x slice           (arith.py:58-71)
2. all-gather of the *exchange buffer* — per rank one chunk holding its x slice
   followed by its x̂ values, padded to a common length so a single
   ``all_gather_into_tensor`` lands every chunk in place (rank-major)
3. ``UP_TOP``   x̂ of the top levels from the gathered level-p values
4. ``COUPLE``   ŷ_t = Σ_s S^{t,s} x̂_s for t own or top            (arith.py:72-81)
5. ``DOWN``     ŷ pushed down through the transfers into own clusters (arith.py:82-97)
6. ``NEAR``     y_t = Σ_s D_{t,s} x_s + V_t ŷ_t for its own leaves  (arith.py:98-104)

The plan is data: per phase a list of launches, each a list of work items
(≤ 64 output rows) built from segments (an A block of ≤ 32 columns from one of
six payloads times ≤ 32 rows of a vector buffer).  libh2b executes it
(``h2b_plan_*``: grouped complex GEMM on the FP64 tensor pipe for q ≥ 2,
grouped GEMV for q = 1); the CPU tests execute the same plan with a numpy
interpreter to check the partition and exchange logic on gloo.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MM_M, MM_K = 64, 32
PH_UP_OWN, PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR = 0, 1, 2, 3, 4
PH_LEAFBACK = 5  # leaf back-transform alone (accumulating), after the fast q=1 near-field
PHASES = (PH_UP_OWN, PH_UP_TOP, PH_COUPLE, PH_DOWN, PH_NEAR)
PAY_VT, PAY_TT, PAY_T, PAY_S, PAY_D, PAY_V = 0, 1, 2, 3, 4, 5
N_PAY = 6
B_X, B_XHAT, B_YHAT, B_Y = 0, 1, 2, 3
ITEM_ACC, ITEM_BCAST = 256, 512
SEG_TRANS, SEG_GATHER = 256, 512


@dataclass
class Partition:
    """Row/skeleton ownership and the exchange-buffer layout shared by all ranks."""

    G: int
    p: int                  # partition level, G = 2**p
    roots: np.ndarray       # [G] packed index of each rank's level-p cluster
    row0: np.ndarray        # [G] first permuted row of each rank
    nrows: np.ndarray       # [G] rows of each rank
    owner: np.ndarray       # [P] owning rank of each cluster (-1: top level, computed by all)
    hat: np.ndarray         # [P] exchange-buffer row of x̂_c / ŷ_c (-1 when k_c = 0)
    chunk: int              # rows per rank chunk: nmax (x slice) + kmax (own x̂)
    nmax: int
    xlen: int               # G * chunk + Σ k over top clusters

    def xrow(self, i):
        """Exchange-buffer row of permuted point i."""
        g = int(np.searchsorted(self.row0, i, side="right") - 1)
        return g * self.chunk + (i - int(self.row0[g]))


def _with_far(pk, far):
    import dataclasses
    return dataclasses.replace(pk, **far)


def partition(pk, G: int) -> Partition:
    if G < 1 or (G & (G - 1)):
        raise ValueError("the subtree partition needs a power-of-two number of ranks")
    p = G.bit_length() - 1
    P = pk.num_clusters
    lev = pk.c_level
    min_leaf = int(lev[pk.c_child_lo < 0].min())
    if p > min_leaf or int(pk.level_ptr[p + 1] - pk.level_ptr[p]) != G:
        raise ValueError(f"{G} ranks need {G} clusters on level {p} above every leaf")
    roots = np.arange(pk.level_ptr[p], pk.level_ptr[p + 1], dtype=np.int64)
    owner = np.full(P, -1, dtype=np.int64)
    owner[roots] = np.arange(G)
    for lvl in range(p + 1, pk.depth):  # parents precede children level by level
        for c in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            owner[c] = owner[pk.c_parent[c]]
    row0 = pk.c_start[roots].astype(np.int64)
    nrows = pk.c_size[roots].astype(np.int64)
    kown = np.zeros(G, dtype=np.int64)
    local = np.full(P, -1, dtype=np.int64)
    for c in range(P):  # level-major order inside each rank
        if owner[c] >= 0 and pk.c_rank[c] > 0:
            local[c] = kown[owner[c]]
            kown[owner[c]] += pk.c_rank[c]
    nmax = int(nrows.max())
    nmax += nmax & 1  # even: x rows of every leaf stay 32-byte aligned (256-bit loads)
    chunk = nmax + int(kown.max())
    chunk += chunk & 1
    hat = np.full(P, -1, dtype=np.int64)
    own = local >= 0
    hat[own] = owner[own] * chunk + nmax + local[own]
    t = G * chunk
    for c in range(P):
        if owner[c] < 0 and pk.c_rank[c] > 0:
            hat[c] = t
            t += int(pk.c_rank[c])
    return Partition(G=G, p=p, roots=roots, row0=row0, nrows=nrows, owner=owner, hat=hat,
                     chunk=chunk, nmax=nmax, xlen=t)


@dataclass
class ShardPlan:
    rank: int
    part: Partition
    payloads: list                          # N_PAY complex128 arrays
    phases: dict = field(default_factory=dict)  # phase -> (launch_counts, items, segs)
    gather: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))  # gathered B rows
    near_fast: dict | None = None  # q=1 near-field work lists for the streaming kernel
    couple_fast: dict | None = None  # q=1 coupling work lists for the panel kernels
    fills: dict | None = None  # device-generated payloads (sizes + block descriptors)

    @property
    def row0(self):
        return int(self.part.row0[self.rank])

    @property
    def nrows(self):
        return int(self.part.nrows[self.rank])

    def payload_sizes(self):
        """Complex elements of each payload (described blocks included)."""
        if self.fills is not None:
            return list(self.fills["sizes"])
        return [int(a.size) for a in self.payloads]

    def payload_bytes(self):
        return 16 * int(sum(self.payload_sizes()))


class _Builder:
    def __init__(self):
        from ._abi import MM_ITEM, MM_SEG
        self._it, self._sg = MM_ITEM, MM_SEG
        self.items, self.segs, self.counts = [], [], []
        self._first = 0

    def seg(self, a_src, a_off, lda, m0, k, b_src, b_row, gather=False, trans=False):
        """K-chunks of one A block: row-major A[i][j] = p[a_off + (m0+i)*lda + j], or transposed
        (A[i][j] = p[a_off + j*lda + m0 + i])."""
        for k0 in range(0, k, MM_K):
            off = a_off + (k0 * lda + m0 if trans else m0 * lda + k0)
            self.segs.append((off, b_row + k0, min(MM_K, k - k0), lda,
                              a_src | (b_src << 4) | (SEG_GATHER if gather else 0)
                              | (SEG_TRANS if trans else 0), 0))

    def begin(self):
        return len(self.segs)

    def end(self, s0, c_row, m, dst, acc=False):
        self.items.append((c_row, m, s0, len(self.segs) - s0, dst | (ITEM_ACC if acc else 0), 0))

    def launch(self):
        n = len(self.items) - self._first
        if n:
            self.counts.append(n)
        self._first = len(self.items)

    def done(self):
        self.launch()
        return (np.asarray(self.counts, dtype=np.int64),
                np.array(self.items, dtype=self._it), np.array(self.segs, dtype=self._sg))


class _GBlock:
    """A payload block not materialised on the host: rows x cols of global section `sec` at
    element `g0` (row-major), to be written as-is or transposed by the device generator."""

    def __init__(self, sec, g0, rows, cols, trans=False):
        self.sec, self.g0, self.rows, self.cols, self.trans = sec, int(g0), int(rows), int(cols), trans

    @property
    def T(self):
        return _GBlock(self.sec, self.g0, self.rows, self.cols, not self.trans)

    @property
    def size(self):
        return self.rows * self.cols


class _NBlock:
    """A near-field block sampled on the device: rows of leaf t, columns of leaf s."""

    def __init__(self, t0, nt, s0, ns):
        self.t0, self.nt, self.s0, self.ns = int(t0), int(nt), int(s0), int(ns)
        self.size = self.nt * self.ns


SEC_V, SEC_T, SEC_S = 0, 1, 2  # global sections of the synthetic generator (= libh2b H2B_SEC_*)


def plan_shard(pk, G: int, g: int, part: Partition | None = None, bcast: bool = False,
               couple_panels: bool = False, device_payloads: bool = False) -> ShardPlan:
    """Payloads and work lists of rank g of G (see the module docstring).

    ``bcast``: the UP_OWN items also store their x̂ rows into every peer's exchange buffer
    (P2P stores over NVLink, libh2b ITEM_BCAST) — the all-gather of x̂ fused into the kernel that
    computes it; the x slice is pushed by ``h2b_plan_bcast_rows``.
    ``couple_panels``: each coupling row as one panel against gathered x̂ rows (full K chunks,
    for multi-RHS use) instead of one segment per source block.
    ``device_payloads``: payloads the host does not hold (structure-exact operators: seeded far
    field, near-field from geometry) are described, not materialised — the rank's device fills
    them (libh2b h2b_plan_fill_synthetic / _near) with the values the single-GPU operator has."""
    part = part or partition(pk, G)
    if not 0 <= g < G:
        raise ValueError("rank out of range")
    own = part.owner == g
    top = part.owner < 0
    mine = own | top
    k = pk.c_rank.astype(np.int64)
    lo_of, hi_of = pk.c_child_lo, pk.c_child_hi
    hat = part.hat
    pays = [[] for _ in range(N_PAY)]
    size = [0] * N_PAY
    synth_fills = [[] for _ in range(N_PAY)]  # {plan_off, global_off, rows, cols, trans, sec}
    near_fills = []                          # {plan_off, t_start, nt, s_start, ns}
    far_dev = device_payloads and pk.sbuf.size == 0 and pk.vbuf.size == 0 and "synthetic" in pk.meta
    near_dev = device_payloads and pk.dbuf.size == 0 and "geometry" in pk.meta
    if not far_dev and pk.sbuf.size == 0 and pk.vbuf.size == 0 and "synthetic" in pk.meta:
        from .synthetic import host_far_field  # CPU engines: the same values, on the host
        pk = _with_far(pk, host_far_field(pk))

    def put(which, mat):
        off = size[which]
        if isinstance(mat, _GBlock):
            synth_fills[which].append((off, mat.g0, mat.rows, mat.cols, int(mat.trans), mat.sec))
        elif isinstance(mat, _NBlock):
            near_fills.append((off, mat.t0, mat.nt, mat.s0, mat.ns))
        else:
            pays[which].append(np.ascontiguousarray(mat, dtype=np.complex128).ravel())
        size[which] += mat.size
        return off

    def xrow_leaf(c):
        o = int(part.owner[c])
        return o * part.chunk + int(pk.c_start[c]) - int(part.row0[o])

    def V(c):
        n, kc = int(pk.c_size[c]), int(k[c])
        if far_dev:
            return _GBlock(SEC_V, pk.c_v_off[c], n, kc)
        return pk.vbuf[pk.c_v_off[c]:pk.c_v_off[c] + n * kc].reshape(n, kc)

    def T(c):
        m = int(k[lo_of[c]] + k[hi_of[c]])
        if far_dev:
            return _GBlock(SEC_T, pk.c_t_off[c], m, int(k[c]))
        return pk.tbuf[pk.c_t_off[c]:pk.c_t_off[c] + m * k[c]].reshape(m, int(k[c]))

    def S(b, kt, ks):
        if far_dev:
            return _GBlock(SEC_S, pk.s_off[b], kt, ks)
        return pk.sbuf[pk.s_off[b]:pk.s_off[b] + kt * ks].reshape(kt, ks)

    def up(Bd, levels, sel):
        for lvl in levels:
            for c in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
                if not sel[c] or k[c] == 0:
                    continue
                kc = int(k[c])
                if lo_of[c] < 0:
                    n = int(pk.c_size[c])
                    off = put(PAY_VT, V(c).T)
                    for m0 in range(0, kc, MM_M):
                        s0 = Bd.begin()
                        Bd.seg(PAY_VT, off, n, m0, n, B_X, xrow_leaf(c))
                        Bd.end(s0, hat[c] + m0, min(MM_M, kc - m0), B_XHAT)
                else:
                    lo, hi = int(lo_of[c]), int(hi_of[c])
                    klo, khi = int(k[lo]), int(k[hi])
                    off = put(PAY_TT, T(c).T) if klo + khi else 0
                    for m0 in range(0, kc, MM_M):
                        s0 = Bd.begin()
                        if klo:
                            Bd.seg(PAY_TT, off, klo + khi, m0, klo, B_XHAT, hat[lo])
                        if khi:
                            Bd.seg(PAY_TT, off + klo, klo + khi, m0, khi, B_XHAT, hat[hi])
                        Bd.end(s0, hat[c] + m0, min(MM_M, kc - m0), B_XHAT)
            Bd.launch()

    phases = {}
    Bd = _Builder()
    up(Bd, range(pk.depth - 1, part.p - 1, -1), own)
    phases[PH_UP_OWN] = Bd.done()
    if bcast:
        phases[PH_UP_OWN][1]["flags"] |= ITEM_BCAST
    Bd = _Builder()
    up(Bd, range(part.p - 1, -1, -1), top)
    phases[PH_UP_TOP] = Bd.done()

    Bd = _Builder()  # coupling: every own/top target with k > 0 (zero when it has no block)
    # payload 3 holds, per target, the stacked transposed panel [S_t,s1ᵀ; S_t,s2ᵀ; ...]
    # ((Σ k_s) x k_t, the single-GPU layout): the q = 1 panel kernels read it with gathered x̂
    # rows, the grouped kernels as transposed segments (one per source, or one gathered panel)
    gat, n_gat = [], 0            # gathered x̂ rows (panel mode)
    cf_items, cf_xcol, n_xcol = [], [], 0
    for t in np.nonzero(mine & (k > 0))[0]:
        kt = int(k[t])
        blocks = []
        for b in range(pk.s_row_ptr[t], pk.s_row_ptr[t + 1]):
            s = int(pk.s_col[b])
            if k[s] == 0:
                continue
            blocks.append((S(b, kt, int(k[s])), s))
        R = int(sum(k[s] for _, s in blocks))
        panel = size[PAY_S]
        for B, _ in blocks:  # contiguous: the stacked panel [S_t,s1ᵀ; S_t,s2ᵀ; ...]
            put(PAY_S, B.T)
        rows = [np.arange(hat[s], hat[s] + k[s]) for _, s in blocks]
        cf_items.append((panel, n_xcol, int(hat[t]), R, kt))
        cf_xcol.extend(rows)
        n_xcol += R
        for m0 in range(0, kt, MM_M):
            s0 = Bd.begin()
            if couple_panels and R:
                Bd.seg(PAY_S, panel, kt, m0, R, B_XHAT, n_gat, gather=True, trans=True)
            else:
                r = 0
                for B, s in blocks:
                    ks = int(k[s])
                    Bd.seg(PAY_S, panel + r * kt, kt, m0, ks, B_XHAT, hat[s], trans=True)
                    r += ks
            Bd.end(s0, hat[t] + m0, min(MM_M, kt - m0), B_YHAT)
        if couple_panels and R:
            gat.extend(rows)
            n_gat += R
    phases[PH_COUPLE] = Bd.done()
    gather = (np.concatenate(gat).astype(np.int32) if gat else np.zeros(0, np.int32))
    from ._abi import COUPLE_ITEM
    couple_fast = dict(items=np.array(cf_items, dtype=COUPLE_ITEM),
                       xcol=(np.concatenate(cf_xcol).astype(np.int32) if cf_xcol
                             else np.zeros(0, np.int32)))

    Bd = _Builder()  # downward, root first: [ŷ_lo; ŷ_hi] += [T_lo; T_hi] ŷ_c
    for lvl in range(pk.depth - 1):
        for c in range(pk.level_ptr[lvl], pk.level_ptr[lvl + 1]):
            if not mine[c] or k[c] == 0 or lo_of[c] < 0:
                continue
            lo, hi = int(lo_of[c]), int(hi_of[c])
            klo, khi, kc = int(k[lo]), int(k[hi]), int(k[c])
            if klo + khi == 0 or not (mine[lo] or mine[hi]):
                continue
            off = put(PAY_T, T(c))
            for ch, r0, kch in ((lo, 0, klo), (hi, klo, khi)):
                if not mine[ch] or kch == 0:
                    continue
                for m0 in range(0, kch, MM_M):
                    s0 = Bd.begin()
                    Bd.seg(PAY_T, off + r0 * kc, kc, m0, kc, B_YHAT, hat[c])
                    Bd.end(s0, hat[ch] + m0, min(MM_M, kch - m0), B_YHAT, acc=True)
        Bd.launch()
    phases[PH_DOWN] = Bd.done()

    Bd = _Builder()  # near-field + leaf back-transform of own leaves -> local y rows
    r0 = int(part.row0[g])
    near_blocks, v_offs = {}, {}
    sample = None
    if pk.dbuf.size == 0 and pk.n_near and not near_dev:  # not on the host: sample this rank's rows
        from .nearfield import assemble_block, geometry_arrays
        geo = geometry_arrays(pk.meta["geometry"])
        sample = lambda rows, cols: assemble_block(*geo, rows, cols)  # noqa: E731
    for t in np.nonzero(own & (lo_of < 0))[0]:
        nt = int(pk.c_size[t])
        blocks = []
        if sample is not None:
            rows = pk.perm[pk.c_start[t]:pk.c_start[t] + nt]
            srcs = pk.d_col[pk.d_row_ptr[t]:pk.d_row_ptr[t + 1]]
            panel = sample(rows, np.concatenate([pk.perm[pk.c_start[s]:pk.c_start[s] + pk.c_size[s]]
                                                 for s in srcs]))
        c0 = 0
        for b in range(pk.d_row_ptr[t], pk.d_row_ptr[t + 1]):
            s = int(pk.d_col[b])
            ns = int(pk.c_size[s])
            if near_dev:
                D = _NBlock(pk.c_start[t], nt, pk.c_start[s], ns)
            elif sample is not None:
                D = panel[:, c0:c0 + ns]
                c0 += ns
            else:
                D = pk.dbuf[pk.d_off[b]:pk.d_off[b] + nt * ns].reshape(nt, ns)
            blocks.append((put(PAY_D, D), s, ns))
        near_blocks[t] = [(off, xrow_leaf(s)) for off, s, _ in blocks]
        voff = put(PAY_V, V(t)) if k[t] > 0 else -1
        v_offs[t] = voff
        for m0 in range(0, nt, MM_M):
            s0 = Bd.begin()
            for off, s, ns in blocks:
                Bd.seg(PAY_D, off, ns, m0, ns, B_X, xrow_leaf(s))
            if voff >= 0:
                Bd.seg(PAY_V, voff, int(k[t]), m0, int(k[t]), B_YHAT, hat[t])
            Bd.end(s0, int(pk.c_start[t]) - r0 + m0, min(MM_M, nt - m0), B_Y)
    phases[PH_NEAR] = Bd.done()

    # q = 1: the same near-field on the streaming kernel (uniform 32/64-point leaves), the leaf
    # back-transform as its own accumulating phase
    own_leaves = np.nonzero(own & (lo_of < 0))[0]
    sizes = {int(pk.c_size[t]) for t in own_leaves}
    for t in own_leaves:
        sizes.update(int(pk.c_size[s]) for s in pk.d_col[pk.d_row_ptr[t]:pk.d_row_ptr[t + 1]])
    near_fast = None
    Bd = _Builder()
    for t in own_leaves:
        if k[t] > 0:
            nt = int(pk.c_size[t])
            for m0 in range(0, nt, MM_M):
                s0 = Bd.begin()
                Bd.seg(PAY_V, v_offs[t], int(k[t]), m0, int(k[t]), B_YHAT, hat[t])
                Bd.end(s0, int(pk.c_start[t]) - r0 + m0, min(MM_M, nt - m0), B_Y, acc=True)
    phases[PH_LEAFBACK] = Bd.done()
    if len(sizes) == 1 and sizes.pop() in (32, 64) and len(own_leaves):
        from ._abi import NEAR_BLK, NEAR_ITEM
        ns = int(pk.c_size[own_leaves[0]])
        avg = np.mean([len(near_blocks[t]) for t in own_leaves])
        R = 1
        while R < 4 and R * 128 // (ns // 2) * ns * 16.0 * avg < 24e3:
            R *= 2
        rb = R * 128 // (ns // 2)
        items, blks = [], []
        for t in own_leaves:
            first = len(blks)
            blks.extend(near_blocks[t])
            for row0 in range(0, ns, rb):
                items.append((int(pk.c_start[t]) - r0 + row0, first, len(near_blocks[t]), row0, 0))
        near_fast = dict(items=np.array(items, dtype=NEAR_ITEM), blks=np.array(blks, dtype=NEAR_BLK),
                         ns=ns, R=R)

    payloads = [np.concatenate(a) if a else np.zeros(0, np.complex128) for a in pays]
    deferred = any(synth_fills) or bool(near_fills)
    if deferred:
        # sections the device fills carry sizes only; sections built from host arrays (e.g. the
        # reference-built far field of an operator whose near-field is sampled on the device)
        # keep their data — a section is never mixed (far / near payloads are all-or-nothing)
        for i in range(N_PAY):
            dev_filled = bool(synth_fills[i]) or (i == PAY_D and bool(near_fills))
            if dev_filled:
                assert not pays[i], "payload section mixes host data and device fills"
                payloads[i] = np.zeros(0, np.complex128)
    fills = None
    if deferred:
        fills = dict(sizes=list(size),
                     synth=[np.array(f, dtype=np.int64).reshape(-1, 6) for f in synth_fills],
                     near=np.array(near_fills, dtype=np.int64).reshape(-1, 5),
                     seed=int(pk.meta.get("synthetic", {}).get("seed", 0)),
                     geometry=pk.meta.get("geometry"), perm=pk.perm if near_fills else None)
    return ShardPlan(rank=g, part=part, payloads=payloads, phases=phases, gather=gather,
                     near_fast=near_fast, couple_fast=couple_fast, fills=fills)
