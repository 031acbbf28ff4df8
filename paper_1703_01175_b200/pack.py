"""Level-packed structure-of-arrays form of an H² operator (the upload format).

The reference keeps its operator as Python dicts of small numpy blocks
(`H2Matrix`, /root/reference/pkg/src/h2vie/build.py:135-187;
`NestedBasis`, build.py:65-132; `ClusterTree`, clustering.py:48-117).
`pack_h2` flattens one such object, once, into a handful of flat arrays that
the CUDA side consumes as-is:

* clusters are renumbered *level-major*: packed index ``p = level_ptr[l] + i``
  where ``i`` is the position of the cluster in ``tree.levels[l]``
  (clustering.py:64-67).  The reference cluster id is kept in ``c_id``.
* per-cluster int tables: start/size in the permuted index space, rank k
  (``basis.rank``, build.py:76), level, children, parent (packed indices,
  -1 when absent), skeleton offset ``c_xhat_off`` (prefix sum of k, so x̂ and
  ŷ are flat K-long buffers).
* payloads are complex128, row-major (C order), unpadded and concatenated:

  - ``vbuf``: leaf bases V_c (n_c x k_c) at ``c_v_off[p]`` (build.py:79-81)
  - ``tbuf``: transfer pair T_lo (k_lo x k_c) then T_hi (k_hi x k_c) at
    ``c_t_off[p]`` (build.py:83-85)
  - ``sbuf``: couplings S^{t,s} (k_t x k_s), CSR by packed target index
    (``s_row_ptr``/``s_col``/``s_off``), rows in packed order, columns in the
    sorted ``btree.admissible`` order (clustering.py:188)
  - ``dbuf``: near-field D_{t,s} (n_t x n_s), CSR by packed target leaf
    (``d_row_ptr``/``d_col``/``d_off``), sorted ``btree.inadmissible`` order
    (build.py:321-324).  The blocks of one target leaf are contiguous, so each
    leaf's near-field row panel is one contiguous byte range.

Payload offsets are int64 (config 4's near-field alone is ~7e9 elements).

The same object round-trips to disk (`save_packed` / `load_packed`): the
reference has no serialisation of `H2Matrix`, and operators of
the BASELINE sizes take minutes to hours to build, so they are built once in a
container that has the reference and replayed everywhere else.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field, fields

import numpy as np

FORMAT_VERSION = 1

_INT_TABLES = (
    "level_ptr", "c_start", "c_size", "c_rank", "c_level", "c_child_lo",
    "c_child_hi", "c_parent", "c_id", "c_xhat_off", "c_v_off", "c_t_off",
    "s_row_ptr", "s_col", "s_off", "d_row_ptr", "d_col", "d_off", "perm",
)
_PAYLOADS = ("vbuf", "tbuf", "sbuf", "dbuf")


@dataclass
class PackedH2:
    n: int
    depth: int
    level_ptr: np.ndarray      # int32[depth+1]
    c_start: np.ndarray        # int32[P]
    c_size: np.ndarray         # int32[P]
    c_rank: np.ndarray         # int32[P]
    c_level: np.ndarray        # int32[P]
    c_child_lo: np.ndarray     # int32[P]  packed index or -1
    c_child_hi: np.ndarray     # int32[P]
    c_parent: np.ndarray       # int32[P]
    c_id: np.ndarray           # int32[P]  reference cluster id
    c_xhat_off: np.ndarray     # int64[P+1] prefix sum of ranks
    c_v_off: np.ndarray        # int64[P]  -1 for non-leaves
    c_t_off: np.ndarray        # int64[P]  -1 for leaves
    s_row_ptr: np.ndarray      # int64[P+1]
    s_col: np.ndarray          # int32[nS] packed source index
    s_off: np.ndarray          # int64[nS]
    d_row_ptr: np.ndarray      # int64[P+1]
    d_col: np.ndarray          # int32[nD] packed source leaf index
    d_off: np.ndarray          # int64[nD]
    perm: np.ndarray           # int64[N] (clustering.py:63,86)
    vbuf: np.ndarray           # complex128
    tbuf: np.ndarray
    sbuf: np.ndarray
    dbuf: np.ndarray
    meta: dict = field(default_factory=dict)

    # ------------------------------------------------------------------
    @property
    def num_clusters(self):
        return int(self.c_start.size)

    @property
    def total_rank(self):
        return int(self.c_xhat_off[-1])

    @property
    def n_coupling(self):
        return int(self.s_col.size)

    @property
    def n_near(self):
        return int(self.d_col.size)

    def is_leaf(self, p):
        return self.c_child_lo[p] < 0

    def leaves(self):
        return np.nonzero(self.c_child_lo < 0)[0]

    def admissible_pairs(self):
        """(t, s) reference-id pairs in CSR order (== sorted btree.admissible)."""
        rows = np.repeat(np.arange(self.num_clusters), np.diff(self.s_row_ptr))
        return self._id_pairs(rows, self.s_col)

    def inadmissible_pairs(self):
        rows = np.repeat(np.arange(self.num_clusters), np.diff(self.d_row_ptr))
        return self._id_pairs(rows, self.d_col)

    def _id_pairs(self, rows, cols):
        t = self.c_id[rows].astype(np.int64)
        s = self.c_id[cols].astype(np.int64)
        order = np.lexsort((s, t))
        return list(zip(t[order].tolist(), s[order].tolist()))

    def element_counts(self):
        """E_V, E_T, E_S, E_D and K of SURVEY.md §8(d)."""
        if self.sbuf.size or self.vbuf.size or self.tbuf.size:
            ev, et, es = int(self.vbuf.size), int(self.tbuf.size), int(self.sbuf.size)
        else:  # far field not materialised on the host (filled on the device)
            ev, et, es = self.far_elems_expected()
        return dict(E_V=ev, E_T=et, E_S=es, E_D=self.d_elems_expected(), K=self.total_rank)

    def storage_bytes(self):
        """Same total as H2Matrix.storage_bytes() (build.py:176-187)."""
        return int(self.perm.nbytes + 16 * (self.vbuf.size + self.tbuf.size
                                            + self.sbuf.size + self.d_elems_expected()))

    def algorithmic_bytes(self, q=1):
        """B_alg(q) = 16(E_V+E_T+E_S+E_D) + 32 q (N + K)."""
        e = self.element_counts()
        return 16 * (e["E_V"] + e["E_T"] + e["E_S"] + e["E_D"]) + 32 * q * (self.n + e["K"])

    def d_elems_expected(self):
        """Near-field elements implied by the tables: sum n_t * n_s over inadmissible pairs."""
        rows = np.repeat(np.arange(self.num_clusters), np.diff(self.d_row_ptr))
        return int(np.sum(self.c_size[rows].astype(np.int64) * self.c_size[self.d_col].astype(np.int64)))

    def far_elems_expected(self):
        """(E_V, E_T, E_S) implied by the tables (sizes of V, T, S even when not materialised)."""
        rank, size = self.c_rank.astype(np.int64), self.c_size.astype(np.int64)
        lo, hi = self.c_child_lo, self.c_child_hi
        leaf = lo < 0
        ev = int(np.sum(size[leaf] * rank[leaf]))
        nl = ~leaf
        et = int(np.sum((rank[lo[nl]] + rank[hi[nl]]) * rank[nl]))
        rows = np.repeat(np.arange(self.num_clusters), np.diff(self.s_row_ptr))
        es = int(np.sum(rank[rows] * rank[self.s_col]))
        return ev, et, es

    def near_bytes(self, q=1):
        """Algorithmic bytes of the near-field phase alone: D once, x_s and y_t once."""
        return 16 * self.d_elems_expected() + 32 * q * self.n

    def flops(self, q=1):
        """F(q) = 8 q (2E_V + 2E_T + E_S + E_D)."""
        e = self.element_counts()
        return 8 * q * (2 * e["E_V"] + 2 * e["E_T"] + e["E_S"] + e["E_D"])


# ----------------------------------------------------------------------
# packing from a reference H2Matrix (duck-typed: no import of h2vie here)
# ----------------------------------------------------------------------

def pack_h2(h2) -> PackedH2:
    """Flatten a reference ``H2Matrix`` into a `PackedH2`.

    Reads only the public attributes the reference matvec reads
    (arith.py:52-104): tree.levels/clusters/perm/depth, basis.rank/leaf_v/
    transfers, coupling{(t,s)}, dense{(t,s)}.
    """
    tree = h2.tree
    basis = h2.basis
    depth = int(tree.depth)
    level_ptr = np.zeros(depth + 1, dtype=np.int32)
    order = []
    for lvl in range(depth):
        ids = list(tree.levels[lvl])
        order.extend(ids)
        level_ptr[lvl + 1] = level_ptr[lvl] + len(ids)
    P = len(order)
    pidx = {cid: p for p, cid in enumerate(order)}

    def tab(dtype=np.int32, fill=0):
        return np.full(P, fill, dtype=dtype)

    c_start, c_size, c_rank, c_level = tab(), tab(), tab(), tab()
    c_lo, c_hi, c_par = tab(fill=-1), tab(fill=-1), tab(fill=-1)
    c_id = np.asarray(order, dtype=np.int32)
    for p, cid in enumerate(order):
        c = tree.cluster(cid)
        c_start[p] = c.start
        c_size[p] = c.stop - c.start
        c_rank[p] = basis.rank(cid)
        c_level[p] = c.level
        if not c.is_leaf:
            c_lo[p] = pidx[c.child_lo]
            c_hi[p] = pidx[c.child_hi]
        if c.parent >= 0:
            c_par[p] = pidx[c.parent]
    c_xhat_off = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(c_rank, out=c_xhat_off[1:])

    # leaf bases and transfers
    c_v_off = np.full(P, -1, dtype=np.int64)
    c_t_off = np.full(P, -1, dtype=np.int64)
    vparts, tparts = [], []
    voff = toff = 0
    for p, cid in enumerate(order):
        k = int(c_rank[p])
        if c_lo[p] < 0:
            c_v_off[p] = voff
            if k > 0:
                v = np.ascontiguousarray(basis.leaf_v[cid], dtype=np.complex128)
                assert v.shape == (c_size[p], k)
                vparts.append(v.ravel())
                voff += v.size
        else:
            c_t_off[p] = toff
            if k > 0:
                t_lo, t_hi = basis.transfers[cid]
                assert t_lo.shape == (c_rank[c_lo[p]], k) and t_hi.shape == (c_rank[c_hi[p]], k)
                for t in (t_lo, t_hi):
                    t = np.ascontiguousarray(t, dtype=np.complex128)
                    tparts.append(t.ravel())
                    toff += t.size

    def csr(blocks, shape_of):
        rows = {}
        for (t, s) in blocks:
            rows.setdefault(pidx[t], []).append((t, s))
        row_ptr = np.zeros(P + 1, dtype=np.int64)
        cols, offs, parts = [], [], []
        off = 0
        for p in range(P):
            items = sorted(rows.get(p, []), key=lambda ts: ts[1])
            row_ptr[p + 1] = row_ptr[p] + len(items)
            for (t, s) in items:
                m = np.ascontiguousarray(blocks[(t, s)], dtype=np.complex128)
                assert m.shape == shape_of(t, s), (m.shape, shape_of(t, s))
                cols.append(pidx[s])
                offs.append(off)
                parts.append(m.ravel())
                off += m.size
        buf = np.concatenate(parts) if parts else np.zeros(0, np.complex128)
        return (row_ptr, np.asarray(cols, dtype=np.int32),
                np.asarray(offs, dtype=np.int64), buf)

    s_row_ptr, s_col, s_off, sbuf = csr(
        h2.coupling, lambda t, s: (basis.rank(t), basis.rank(s)))
    d_row_ptr, d_col, d_off, dbuf = csr(
        h2.dense, lambda t, s: (tree.cluster(t).size, tree.cluster(s).size))

    meta = dict(format=FORMAT_VERSION, eps_acc=float(getattr(h2.params, "eps_acc", 0.0)),
                eps_aca=float(getattr(h2.params, "eps_aca", 0.0)))
    return PackedH2(
        n=int(tree.n_points), depth=depth, level_ptr=level_ptr,
        c_start=c_start, c_size=c_size, c_rank=c_rank, c_level=c_level,
        c_child_lo=c_lo, c_child_hi=c_hi, c_parent=c_par, c_id=c_id,
        c_xhat_off=c_xhat_off, c_v_off=c_v_off, c_t_off=c_t_off,
        s_row_ptr=s_row_ptr, s_col=s_col, s_off=s_off,
        d_row_ptr=d_row_ptr, d_col=d_col, d_off=d_off,
        perm=np.ascontiguousarray(tree.perm, dtype=np.int64),
        vbuf=np.concatenate(vparts) if vparts else np.zeros(0, np.complex128),
        tbuf=np.concatenate(tparts) if tparts else np.zeros(0, np.complex128),
        sbuf=sbuf, dbuf=dbuf, meta=meta,
    )


def validate(pk: PackedH2):
    """Structural self-checks; raises ValueError on a malformed operator."""
    P = pk.num_clusters
    if pk.level_ptr[-1] != P or pk.level_ptr[0] != 0:
        raise ValueError("level_ptr does not cover the clusters")
    if pk.perm.shape != (pk.n,) or not np.array_equal(np.sort(pk.perm), np.arange(pk.n)):
        raise ValueError("perm is not a permutation of 0..N-1")
    leaves = pk.leaves()
    cover = np.zeros(pk.n, dtype=np.int64)
    for p in leaves:
        cover[pk.c_start[p]:pk.c_start[p] + pk.c_size[p]] += 1
    if not np.all(cover == 1):
        raise ValueError("leaves do not tile [0, N)")
    # tiling checksum: sum #t*#s over all blocks == N^2 (clustering.py:218-223)
    tot = 0
    for ptr, col in ((pk.s_row_ptr, pk.s_col), (pk.d_row_ptr, pk.d_col)):
        rows = np.repeat(np.arange(P), np.diff(ptr))
        tot += int(np.sum(pk.c_size[rows].astype(np.int64) * pk.c_size[col].astype(np.int64)))
    if tot != pk.n * pk.n:
        raise ValueError(f"blocks do not tile the index square ({tot} != {pk.n}^2)")
    for p in np.nonzero(np.diff(pk.d_row_ptr))[0]:
        if pk.c_child_lo[p] >= 0:
            raise ValueError("near-field block on a non-leaf target")
    return True


# ----------------------------------------------------------------------
# on-disk format: one uncompressed .npz (arrays) with a JSON header entry
# ----------------------------------------------------------------------

def save_packed(pk: PackedH2, path, extra=None, geometry=None):
    """Write `pk` (+ extras).  With ``geometry`` (a `nearfield.geometry_arrays`
    record) the near-field payload is NOT written: `load_packed` re-assembles it
    from the geometry (nearfield.py), which keeps committed fixtures small."""
    names = _INT_TABLES + (_PAYLOADS if geometry is None else _PAYLOADS[:3])
    arrays = {name: getattr(pk, name) for name in names}
    head = dict(n=pk.n, depth=pk.depth, meta=pk.meta, version=FORMAT_VERSION)
    if geometry is not None:
        head["geometry"] = geometry
    arrays["__header__"] = np.frombuffer(json.dumps(head).encode(), dtype=np.uint8)
    for k, v in (extra or {}).items():
        arrays["extra__" + k] = np.asarray(v)
    tmp = str(path) + ".tmp.npz"
    np.savez(tmp, **arrays)
    os.replace(tmp, path)


def save_structure(pk: PackedH2, path, geometry, seed=0, note="", compact=False):
    """Write only the index tables + geometry of `pk` (a *structure-exact* operator file).

    `load_packed` fills the far-field payloads (V, T, S) with seeded random values of exactly
    the reference shapes and re-assembles the near-field from the geometry: same bytes, flops
    and block structure as the reference-built operator, for throughput measurements of
    operators too large to ship ("configs 3-5 without a reference build")."""
    arrays = {name: getattr(pk, name) for name in _INT_TABLES if not (compact and name in _DERIVED)}
    head = dict(n=pk.n, depth=pk.depth, meta=pk.meta, version=FORMAT_VERSION, geometry=geometry,
                synthetic=dict(seed=int(seed), note=note))
    arrays["__header__"] = np.frombuffer(json.dumps(head).encode(), dtype=np.uint8)
    tmp = str(path) + ".tmp.npz"
    (np.savez_compressed if compact else np.savez)(tmp, **arrays)
    os.replace(tmp, path)


_DERIVED = ("c_xhat_off", "c_v_off", "c_t_off", "s_off", "d_off")


def _derive_offsets(kw):
    """The payload offsets implied by the tables (what the packer writes: V/T/S/D blocks in
    cluster / CSR order, -1 where a cluster has no V or T block); compact structure files omit
    them."""
    rank, size = kw["c_rank"].astype(np.int64), kw["c_size"].astype(np.int64)
    lo, hi = kw["c_child_lo"], kw["c_child_hi"]
    leaf = lo < 0
    P = rank.size

    def excl(v):
        o = np.zeros(v.size, np.int64)
        np.cumsum(v[:-1], out=o[1:])
        return o

    out = {"c_xhat_off": np.concatenate([[0], np.cumsum(rank)]).astype(np.int64)}
    out["c_v_off"] = np.where(leaf, excl(np.where(leaf, size * rank, 0)), -1)
    li, hj = np.where(leaf, 0, lo), np.where(leaf, 0, hi)
    out["c_t_off"] = np.where(leaf, -1, excl(np.where(leaf, 0, (rank[li] + rank[hj]) * rank)))
    rows = np.repeat(np.arange(P), np.diff(kw["s_row_ptr"]))
    out["s_off"] = excl(rank[rows] * rank[kw["s_col"]])
    drows = np.repeat(np.arange(P), np.diff(kw["d_row_ptr"]))
    out["d_off"] = excl(size[drows] * size[kw["d_col"]])
    return out


def _synthetic_far_field(kw, spec):
    """Seeded far-field payloads with the shapes implied by the tables (see save_structure and
    synthetic.py: the same values the device generates)."""
    from .synthetic import SCALES, synth_values
    seed = int(spec.get("seed", 0))
    rank, size, lo, hi = kw["c_rank"].astype(np.int64), kw["c_size"].astype(np.int64), \
        kw["c_child_lo"], kw["c_child_hi"]
    leaf = lo < 0
    ev = int(np.sum(size[leaf] * rank[leaf]))
    nl = ~leaf
    et = int(np.sum((rank[lo[nl]] + rank[hi[nl]]) * rank[nl]))
    P = rank.size
    rows = np.repeat(np.arange(P), np.diff(kw["s_row_ptr"]))
    es = int(np.sum(rank[rows] * rank[kw["s_col"]]))
    return dict(vbuf=synth_values(seed, 0, 0, ev, SCALES[0]), tbuf=synth_values(seed, 1, 0, et, SCALES[1]),
                sbuf=synth_values(seed, 2, 0, es, SCALES[2]))


def load_packed(path, with_extra=False, near_on_host=True, far_on_host=True):
    """Read a packed operator.  A compact file (no near-field payload, a geometry record) gets
    its near-field re-assembled on the host (nearfield.py) — or, with ``near_on_host=False``,
    left empty (``dbuf.size == 0``) for `H2Operator` to generate on the device."""
    z = np.load(path, allow_pickle=False)
    head = json.loads(bytes(z["__header__"]).decode())
    if head.get("version") != FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported packed-H2 format {head.get('version')}")
    kw = {name: z[name] for name in _INT_TABLES + _PAYLOADS if name in z.files}
    if any(name not in kw for name in _DERIVED):  # compact structure file
        kw.update({k: v for k, v in _derive_offsets(kw).items() if k not in kw})
    if "synthetic" in head:
        if far_on_host:
            kw.update(_synthetic_far_field(kw, head["synthetic"]))
        else:  # left empty: H2Operator fills V/T/S on the device (synthetic.py)
            kw.update(vbuf=np.zeros(0, np.complex128), tbuf=np.zeros(0, np.complex128),
                      sbuf=np.zeros(0, np.complex128))
    if "dbuf" not in kw:
        if "geometry" not in head:
            raise ValueError(f"{path}: no near-field payload and no geometry to rebuild it from")
        kw["dbuf"] = np.zeros(0, np.complex128)
    pk = PackedH2(n=int(head["n"]), depth=int(head["depth"]), meta=head.get("meta", {}), **kw)
    if "synthetic" in head:
        pk.meta = dict(pk.meta, synthetic=head["synthetic"])
    if "geometry" in head:
        from .nearfield import assemble_near, geometry_arrays
        pk.meta = dict(pk.meta, geometry=head["geometry"])
        if pk.dbuf.size == 0 and pk.n_near and near_on_host:
            pk.dbuf = assemble_near(pk, *geometry_arrays(head["geometry"]))
    if with_extra:
        extra = {k[len("extra__"):]: z[k] for k in z.files if k.startswith("extra__")}
        return pk, extra
    return pk
