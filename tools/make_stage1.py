"""Stage-I factors of the reference builder (and the geometry) for the device Stage II — test fixtures.

Runs only in the build container (imports the reference).  For each small fixture it rebuilds
the operator exactly as tools/make_golden.py does and stores, next to the packed reference
operator, the reference's Stage-I output `build_all_cluster_ab` (build.py:190-225): per cluster
(PACKED order) the grouped factor A (n_c x r), B (sum over partners of n_s x r, partner blocks in
the reference's partner order) and B^T conj(B) (r x r), plus eps_acc and the reference's Stage-II
ranks.  tests/test_gpu_builder.py builds Stage II on the device from these factors.

Usage: python tools/make_stage1.py
"""
import os
import sys

import numpy as np

REF_SRC = os.environ.get("H2VIE_SRC", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

from h2vie import build, clustering as cl, kernel  # noqa: E402
from h2vie.linalg import CompressionParams  # noqa: E402

from paper_1703_01175_b200.pack import pack_h2, save_packed  # noqa: E402

K0 = 2.0 * np.pi


def dump(name, geom, kp, n_min, tol=1e-4):
    cparams = CompressionParams(tol, tol)
    oracle = kernel.entry_oracle(geom, kp)
    tree = cl.ClusterTree(geom.centers, n_min)
    btree = cl.build_block_tree(tree, 1.0)
    abs_map = build.build_all_cluster_ab(tree, btree, oracle, cparams)
    h2 = build.build_h2(geom, kp, cparams, n_min=n_min, eta=1.0)
    pk = pack_h2(h2)
    pidx = {int(c): p for p, c in enumerate(pk.c_id)}
    P = pk.num_clusters
    r = np.zeros(P, np.int32)
    a_off = np.zeros(P + 1, np.int64)
    b_off = np.zeros(P + 1, np.int64)
    m_off = np.zeros(P + 1, np.int64)
    part_ptr = np.zeros(P + 1, np.int64)
    A, B, M, partners, prow = [], [], [], [], []
    for p in range(P):
        ab = abs_map[int(pk.c_id[p])]
        r[p] = ab.rank
        A.append(np.ascontiguousarray(ab.a).ravel())
        B.append(np.ascontiguousarray(ab.b).ravel())
        M.append(np.ascontiguousarray(ab.btb).ravel())
        a_off[p + 1] = a_off[p] + ab.a.size
        b_off[p + 1] = b_off[p] + ab.b.size
        m_off[p + 1] = m_off[p] + ab.btb.size
        for j, s in enumerate(ab.col_clusters):
            partners.append(pidx[int(s)])
            prow.append(int(ab.col_offsets[j]))  # first row of partner j's block in B
        part_ptr[p + 1] = len(partners)
    extra = dict(s1_rank=r, s1_a=np.concatenate(A) if A else np.zeros(0, complex), s1_a_off=a_off,
                 s1_b=np.concatenate(B), s1_b_off=b_off, s1_m=np.concatenate(M), s1_m_off=m_off,
                 s1_part_ptr=part_ptr, s1_partner=np.asarray(partners, np.int32),
                 s1_prow=np.asarray(prow, np.int64), s1_eps_acc=np.float64(cparams.eps_acc),
                 ref_rank=pk.c_rank.copy(), s1_eps_aca=np.float64(cparams.eps_aca),
                 s1_max_rank=np.int64(cparams.max_rank),
                 # the geometry the entries come from (kernel.py:190-210): a device Stage I samples it
                 geom_centers=np.ascontiguousarray(geom.centers, np.float64),
                 geom_chi=np.ascontiguousarray(np.broadcast_to(kp.eps_r, (pk.n,)) - 1.0, np.complex128),
                 geom_k0=np.float64(kp.k0), geom_volume=np.float64(geom.voxel_volume))
    out = os.path.join(ROOT, "tests", "golden", f"stage1_{name}.npz")
    save_packed(pk, out, extra=extra)
    print(f"{name}: N={pk.n} P={P} Stage-I ranks max {r.max()} -> {out} {os.path.getsize(out) / 1e6:.2f} MB")


if __name__ == "__main__":
    kp_def = kernel.KernelParams(k0=K0)
    dump("rod164", kernel.generate_geometry("rod", [16.4], 10, K0), kp_def, 16)
    h = 1.0 / 16
    dump("cube8", kernel.VoxelGeometry(kernel.lattice_centers(8, 8, 8, h), h ** 3, "cube"),
         kernel.KernelParams(K0, 4.0), 32)
    h = 1.0 / 32
    dump("line2048", kernel.VoxelGeometry(kernel.lattice_centers(2048, 1, 1, h), h ** 3, "line"),
         kernel.KernelParams(K0, 4.0), 32)
