"""Generate golden fixtures and packed BASELINE operators FROM THE REFERENCE.

Runs only in the build container, where the reference package is importable
from /root/reference/pkg/src (it does not exist on the GPU box).  It

1. builds small operators with the reference builder (`h2vie.build.build_h2`,
   build.py:312-325), packs them (`paper_1703_01175_b200.pack.pack_h2`) and
   stores, next to them, outputs of the reference's own hot-path functions on
   seeded inputs:  `h2vie.arith.matvec` (arith.py:108-117),
   `h2vie.arith.matmat_apply` (arith.py:120-130), `h2vie.arith.bicgstab_solve`
   (arith.py:605-689), the dense operator (`kernel.assemble_dense`,
   kernel.py:229-234) and the reference partition lists (tree.perm,
   btree.admissible / inadmissible, tiling_checksum).
   -> tests/golden/<name>.npz   (committed, small)

2. with --configs, builds BASELINE configs 1 and 2 exactly as SURVEY.md §8(d)
   specifies and stores the packed operator plus reference matvec outputs
   -> data/cfg<k>.npz          (git-ignored; travels to the GPU box)

Usage:  python tools/make_golden.py [--small] [--configs 1,2]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

# H2VIE_SRC may point at a scratch copy of the reference with its Cython backend built
# (cp -r /root/reference/pkg /tmp/h2ref && python setup.py build_ext --inplace): same code,
# 2.5-4x faster block assembly for the large configs.
REF_SRC = os.environ.get("H2VIE_SRC", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

from h2vie import arith, build, clustering, kernel  # noqa: E402
from h2vie.linalg import CompressionParams  # noqa: E402

from paper_1703_01175_b200.pack import pack_h2, save_packed, validate  # noqa: E402

K0 = 2.0 * np.pi


def _cvec(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _partition_arrays(h2):
    adm = np.asarray(h2.btree.admissible, dtype=np.int64).reshape(-1, 2)
    inadm = np.asarray(h2.btree.inadmissible, dtype=np.int64).reshape(-1, 2)
    return dict(ref_perm=h2.tree.perm.astype(np.int64), ref_admissible=adm,
                ref_inadmissible=inadm,
                ref_tiling=np.int64(clustering.tiling_checksum(h2.btree, h2.tree)),
                ref_storage_bytes=np.int64(h2.storage_bytes()))


def small_fixture(name, geom, kp, n_min, tol=1e-4, dense=True, seed=7, bicg=True):
    t = time.time()
    h2 = build.build_h2(geom, kp, CompressionParams(tol, tol), n_min=n_min, eta=1.0)
    pk = pack_h2(h2)
    validate(pk)
    rng = np.random.default_rng(seed)
    n = h2.n
    X = _cvec(rng, (n, 4))
    Y = np.stack([arith.matvec(h2, X[:, j]) for j in range(4)], axis=1)
    XM = _cvec(rng, (n, 5))
    YM = arith.matmat_apply(h2, XM)
    YM2 = arith.matmat_apply(h2, XM, col_block=2)
    extra = dict(x=X, y=Y, xm=XM, ym=YM, ym_cb2=YM2, **_partition_arrays(h2))
    extra["zero_out"] = arith.matvec(h2, np.zeros(n))
    if dense:
        extra["dense"] = kernel.assemble_dense(geom, kp)
    if bicg:
        rhs = kernel.plane_wave_rhs(geom, K0, [0, -1, 0])
        for tag, tl in (("e3", 1e-3), ("e6", 1e-6)):
            xs, rep = arith.bicgstab_solve(lambda v: arith.matvec(h2, v), rhs, tol=tl, max_iter=400)
            extra[f"bicg_{tag}_x"] = xs
            extra[f"bicg_{tag}_iters"] = np.int64(rep.iterations)
            extra[f"bicg_{tag}_hist"] = np.asarray(rep.residual_history)
            extra[f"bicg_{tag}_conv"] = np.bool_(rep.converged)
        extra["bicg_rhs"] = rhs
    out = os.path.join(ROOT, "tests", "golden", f"{name}.npz")
    save_packed(pk, out, extra=extra)
    print(f"{name}: N={n} P={pk.num_clusters} depth={pk.depth} K={pk.total_rank} "
          f"adm={pk.n_coupling} inadm={pk.n_near} {os.path.getsize(out)/1e6:.2f} MB "
          f"({time.time()-t:.1f}s)", flush=True)


def make_small():
    kp_def = kernel.KernelParams(k0=K0)
    # the reference suite's own session fixtures (tests/conftest.py:16-32)
    g = kernel.generate_geometry("rod", [16.4], 10, K0)
    small_fixture("rod164", g, kp_def, n_min=16)
    g = kernel.generate_geometry("cube_array", [2, 2, 2], 10, K0)
    small_fixture("cube2", g, kp_def, n_min=32)
    # chi = 0: identity model (tests/test_arith.py:22-25,37-40)
    g = kernel.generate_geometry("rod", [6.4], 10, K0)
    small_fixture("identity", g, kernel.KernelParams(k0=K0, eps_r=1.0), n_min=8, bicg=False)
    # ragged / mixed-level trees (tests/test_clustering.py:110-119)
    rng = np.random.default_rng(1234)
    for n, n_min in ((5, 2), (137, 6)):
        pts = rng.normal(size=(n, 3))
        g = kernel.VoxelGeometry(pts, 1e-3, "random")
        small_fixture(f"random{n}", g, kernel.KernelParams(k0=K0, eps_r=4.0), n_min=n_min, bicg=False)
    # scaled-down BASELINE shapes: cube (cfg1/4/5), line (cfg2), plate (cfg3)
    h = 1.0 / 16
    g = kernel.VoxelGeometry(kernel.lattice_centers(8, 8, 8, h), h ** 3, "cube")
    small_fixture("cube8", g, kernel.KernelParams(K0, 4.0), n_min=32, dense=False)
    h = 1.0 / 32
    g = kernel.VoxelGeometry(kernel.lattice_centers(2048, 1, 1, h), h ** 3, "line")
    small_fixture("line2048", g, kernel.KernelParams(K0, 4.0), n_min=32, dense=False)
    h = 1.0 / 16
    g = kernel.VoxelGeometry(kernel.lattice_centers(32, 32, 1, h), h ** 3, "plate")
    small_fixture("plate32", g, kernel.KernelParams(K0, 4.0), n_min=16, dense=False)
    rng = np.random.default_rng(5)
    g = kernel.VoxelGeometry(kernel.lattice_centers(8, 8, 8, h), h ** 3, "cube")
    small_fixture("cube8_rand_eps", g, kernel.KernelParams(K0, 2.0 + 4.0 * rng.random(512)),
                  n_min=16, dense=False, bicg=False)


def make_config(k, seed=0):
    """BASELINE configs (exact construction)."""
    if k == 1:
        h = 1.0 / 16
        g = kernel.VoxelGeometry(kernel.lattice_centers(16, 16, 16, h), h ** 3, "cube")
        kp, n_min, tol = kernel.KernelParams(K0, 4.0), 32, 1e-4
    elif k == 2:
        h = 1.0 / 32
        g = kernel.VoxelGeometry(kernel.lattice_centers(65536, 1, 1, h), h ** 3, "line")
        kp, n_min, tol = kernel.KernelParams(K0, 4.0), 32, 1e-4
    elif k == 3:
        h = 1.0 / 16
        g = kernel.VoxelGeometry(kernel.lattice_centers(512, 512, 1, h), h ** 3, "plate")
        kp, n_min, tol = kernel.KernelParams(K0, 4.0), 64, 1e-4
    else:
        raise ValueError(k)
    t = time.time()
    h2 = build.build_h2(g, kp, CompressionParams(tol, tol), n_min=n_min, eta=1.0)
    tb = time.time() - t
    pk = pack_h2(h2)
    validate(pk)
    rng = np.random.default_rng(seed)
    x = _cvec(rng, h2.n)
    t = time.time()
    y = arith.matvec(h2, x)
    tm = time.time() - t
    x2 = _cvec(rng, h2.n)
    y2 = arith.matvec(h2, x2)
    extra = dict(x=np.stack([x, x2], 1), y=np.stack([y, y2], 1), build_s=np.float64(tb),
                 ref_matvec_s=np.float64(tm), **_partition_arrays(h2))
    if k == 1:
        # GMRES(30) to 1e-6 on the seeded N(0,1) RHS with the reference matvec
        sys.path.insert(0, ROOT)
        from oracle.krylov_oracle import gmres_solve
        xs, rep = gmres_solve(lambda v: arith.matvec(h2, v), x, tol=1e-6, restart=30, max_iter=2000)
        extra.update(gmres_iters=np.int64(rep.iterations), gmres_hist=np.asarray(rep.residual_history),
                     gmres_x=xs)
        xs, rep = arith.bicgstab_solve(lambda v: arith.matvec(h2, v), x, tol=1e-6, max_iter=1000)
        extra.update(bicg_iters=np.int64(rep.iterations), bicg_hist=np.asarray(rep.residual_history))
    if k == 3:
        # plane wave with seeded incidence (SURVEY.md §8d cfg 3): a FRESH default_rng(0), theta
        # first, then phi; then GMRES(50) to 1e-6 on it with the reference matvec (the oracle
        # restatement; the reference has no GMRES) and scipy's count beside it
        rng3 = np.random.default_rng(0)
        th = np.arccos(rng3.uniform(-1, 1))
        ph = rng3.uniform(0, 2 * np.pi)
        d = np.array([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])
        b = kernel.plane_wave_rhs(g, K0, d)
        extra["rhs_plane_wave"] = b
        extra["incidence"] = d
        if os.environ.get("H2B_CFG3_GMRES"):
            from oracle.krylov_oracle import gmres_solve
            t = time.time()
            xs, rep = gmres_solve(lambda v: arith.matvec(h2, v), b, tol=1e-6, restart=50, max_iter=3000)
            extra.update(gmres_iters=np.int64(rep.iterations), gmres_hist=np.asarray(rep.residual_history),
                         gmres_s=np.float64(time.time() - t))
            print(f"cfg3 oracle GMRES(50): {rep.iterations} it, converged {rep.converged}, "
                  f"{time.time() - t:.0f} s", flush=True)
    os.makedirs(os.path.join(ROOT, "data"), exist_ok=True)
    out = os.path.join(ROOT, "data", f"cfg{k}.npz")
    save_packed(pk, out, extra=extra)
    print(f"cfg{k}: N={h2.n} build {tb:.1f}s ref matvec {tm*1e3:.1f} ms "
          f"B_alg={pk.algorithmic_bytes()/1e6:.2f} MB K={pk.total_rank} -> {out}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--configs", default="")
    a = ap.parse_args()
    if a.small:
        make_small()
    for k in [int(c) for c in a.configs.split(",") if c]:
        make_config(k)
