"""Structure-exact operators for BASELINE configs 4 and 5 ("configs 4/5 without a
reference build"): the reference's own cluster tree and block partition (h2vie.clustering, run
here on the exact geometry), per-cluster ranks taken from the reference-built proxies by cluster
size, seeded far-field values, near-field sampled from the geometry on the device.

Bytes, flops and block structure are those of the reference operator up to the proxy ranks;
there is no parity claim (the reference cannot build these here: SURVEY.md §0 finding 4).

    python tools/make_structures.py 4 5    -> structures/cfg<k>.npz (git-ignored, ships to the box)
"""
import os
import sys
import time

import numpy as np

REF_SRC = os.environ.get("H2VIE_SRC", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)
from h2vie import clustering  # noqa: E402

from paper_1703_01175_b200.nearfield import lattice_centers  # noqa: E402
from paper_1703_01175_b200.pack import PackedH2, save_structure  # noqa: E402

# ranks by cluster size (points), from the reference-built 32^3 proxies:
# tol 1e-3: 64 -> 15, 128 -> 17, 256 -> 18, 512 -> 18; tol 1e-4: 64 -> 23, 128 -> 28, 256 -> 28,
# 512 -> 27; larger clusters (no proxy) grow with their electrical size (assumed, stated)
RANKS = {
    4: {64: 15, 128: 17, 256: 18, 512: 18, 1024: 20, 2048: 24, 4096: 30, 8192: 38, 16384: 48,
        32768: 60, 65536: 75},
    5: {64: 23, 128: 28, 256: 28, 512: 27, 1024: 30, 2048: 36, 4096: 44, 8192: 54, 16384: 66},
}
GEOM = {
    4: dict(kind="lattice", dims=[128, 128, 128], h=1 / 16, eps_r=4.0, k0=2 * np.pi),
    5: dict(kind="lattice", dims=[64, 64, 64], h=1 / 16, eps_r={"uniform": [2.0, 6.0], "seed": 0},
            k0=2 * np.pi),
}


def build(k):
    t0 = time.time()
    g = GEOM[k]
    pts = lattice_centers(*g["dims"], g["h"])
    tree = clustering.ClusterTree(pts, 64)
    bt = clustering.build_block_tree(tree, eta=1.0)
    print(f"cfg{k}: tree+blocks {time.time() - t0:.0f}s, {len(bt.admissible)} adm, "
          f"{len(bt.inadmissible)} inadm", flush=True)
    depth = int(tree.depth)
    order = [cid for lvl in range(depth) for cid in tree.levels[lvl]]
    P = len(order)
    pidx = np.full(max(order) + 1, -1, dtype=np.int64)
    pidx[np.asarray(order)] = np.arange(P)
    level_ptr = np.zeros(depth + 1, dtype=np.int32)
    for lvl in range(depth):
        level_ptr[lvl + 1] = level_ptr[lvl] + len(tree.levels[lvl])
    tab = {n: np.full(P, -1 if n in ("c_child_lo", "c_child_hi", "c_parent") else 0, dtype=np.int32)
           for n in ("c_start", "c_size", "c_rank", "c_level", "c_child_lo", "c_child_hi", "c_parent")}
    adm_targets = set(t for t, _ in bt.admissible) | set(s for _, s in bt.admissible)
    for p, cid in enumerate(order):
        c = tree.cluster(cid)
        tab["c_start"][p], tab["c_size"][p], tab["c_level"][p] = c.start, c.stop - c.start, c.level
        if not c.is_leaf:
            tab["c_child_lo"][p], tab["c_child_hi"][p] = pidx[c.child_lo], pidx[c.child_hi]
        if c.parent >= 0:
            tab["c_parent"][p] = pidx[c.parent]
    # ranks: clusters with an admissible block or below one carry a basis (nested bases)
    need = np.zeros(P, dtype=bool)
    for cid in adm_targets:
        need[pidx[cid]] = True
    for lvl in range(1, depth):  # a child of a cluster with a basis needs one too
        for p in range(level_ptr[lvl], level_ptr[lvl + 1]):
            if need[tab["c_parent"][p]]:
                need[p] = True
    sizes = tab["c_size"]
    table = RANKS[k]
    for p in range(P):
        if need[p]:
            key = min(table, key=lambda s: abs(np.log2(s) - np.log2(max(sizes[p], 1))))
            tab["c_rank"][p] = min(table[key], sizes[p])
    rank = tab["c_rank"].astype(np.int64)
    c_xhat_off = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(rank, out=c_xhat_off[1:])
    leaf = tab["c_child_lo"] < 0
    c_v_off = np.full(P, -1, dtype=np.int64)
    c_t_off = np.full(P, -1, dtype=np.int64)
    ev = np.where(leaf, sizes * rank, 0)
    c_v_off[leaf] = (np.cumsum(ev) - ev)[leaf]
    lo, hi = tab["c_child_lo"], tab["c_child_hi"]
    et = np.where(~leaf, (rank[np.maximum(lo, 0)] + rank[np.maximum(hi, 0)]) * rank, 0)
    c_t_off[~leaf] = (np.cumsum(et) - et)[~leaf]

    def csr(pairs, size_of):
        a = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        t, s = pidx[a[:, 0]], pidx[a[:, 1]]
        o = np.lexsort((s, t))
        t, s = t[o], s[o]
        row_ptr = np.zeros(P + 1, dtype=np.int64)
        np.add.at(row_ptr, t + 1, 1)
        np.cumsum(row_ptr, out=row_ptr)
        sz = size_of(t) * size_of(s)
        off = np.cumsum(sz) - sz
        return row_ptr, s.astype(np.int32), off.astype(np.int64)

    s_row_ptr, s_col, s_off = csr(bt.admissible, lambda c: rank[c])
    d_row_ptr, d_col, d_off = csr(bt.inadmissible, lambda c: sizes[c].astype(np.int64))
    e = np.zeros(0, np.complex128)
    pk = PackedH2(n=int(tree.n_points), depth=depth, level_ptr=level_ptr, c_start=tab["c_start"],
                  c_size=tab["c_size"], c_rank=tab["c_rank"], c_level=tab["c_level"],
                  c_child_lo=tab["c_child_lo"], c_child_hi=tab["c_child_hi"], c_parent=tab["c_parent"],
                  c_id=np.asarray(order, dtype=np.int32), c_xhat_off=c_xhat_off, c_v_off=c_v_off,
                  c_t_off=c_t_off, s_row_ptr=s_row_ptr, s_col=s_col, s_off=s_off, d_row_ptr=d_row_ptr,
                  d_col=d_col, d_off=d_off, perm=np.asarray(tree.perm, dtype=np.int64), vbuf=e, tbuf=e,
                  sbuf=e, dbuf=e, meta={"ranks": "proxy ranks by cluster size (tools/make_structures.py)"})
    E_S = int(np.sum(rank[np.repeat(np.arange(P), np.diff(s_row_ptr))] * rank[s_col]))
    E_D = pk.d_elems_expected()
    print(f"cfg{k}: N={pk.n} P={P} K={int(c_xhat_off[-1])} couplings {16 * E_S / 1e9:.1f} GB, "
          f"near-field {16 * E_D / 1e9:.1f} GB, V {16 * ev.sum() / 1e9:.2f} GB, T {16 * et.sum() / 1e9:.2f} GB",
          flush=True)
    os.makedirs(os.path.join(ROOT, "structures"), exist_ok=True)
    out = os.path.join(ROOT, "structures", f"cfg{k}.npz")
    save_structure(pk, out, g, seed=k, note=f"cfg{k}: reference tree/block partition, proxy ranks, "
                   "seeded V/T/S, near-field sampled on device")
    print(f"  -> {out} {os.path.getsize(out) / 1e6:.1f} MB ({time.time() - t0:.0f}s)", flush=True)


if __name__ == "__main__":
    for k in [int(a) for a in sys.argv[1:]]:
        build(k)
