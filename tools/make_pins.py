"""Reference-built pins for BASELINE configs 3 and 5 at sizes that ship to the GPU box.

Runs only in the build container (imports the reference from H2VIE_SRC or
/root/reference/pkg/src).  The full configs do not fit: cfg3's reference build is
7.1 GB (1.7 GB without its near-field) against the GPU box's 512 MiB snapshot, and
cfg5's needs more host memory than this container has (SURVEY.md §0 finding 4).
So each pin is the largest operator of the config's construction whose compact
file (far field only; near-field re-assembled from the geometry on load, checked
here bit-for-bit against the reference build) fits the push:

* ``plate``: a 2-D plate at 16 points/lambda, eps_r = 4, leaf 64, eta 1, tol 1e-4
  (cfg3's construction on a smaller grid, default 256 x 128).  RHS: the unit
  plane wave of SURVEY.md §8(d) — a FRESH default_rng(0), theta =
  arccos(U(-1, 1)) first, then phi = U(0, 2 pi) — plus two N(0,1) vectors for
  the matvec parity.  Stored reference outputs: arith.matvec on both vectors
  and on the plane wave; the oracle's GMRES(50) to 1e-6 iteration count and
  history on the plane wave (the reference has no GMRES), cross-checked with
  scipy.sparse.linalg.gmres.
* ``cube``: a 3-D cube at 16 points/lambda, eps_r = 2 + 4 U[0,1) per cell from
  default_rng(0) (kernel.py:68-75 accepts arrays), leaf 64, tol 1e-4 (cfg5's
  construction on a smaller grid, default 16 x 16 x 32).  RHS: 64 plane waves,
  directions drawn as in cfg3 from one default_rng(0) stream (theta, phi per
  wave).  Stored: arith.matmat_apply on the 64 waves, arith.matvec on one N(0,1)
  vector, and the oracle's block GMRES(30) to 1e-6 (iterations, history).

Usage:  H2VIE_SRC=/tmp/h2ref/src python tools/make_pins.py plate [nx ny]
        H2VIE_SRC=/tmp/h2ref/src python tools/make_pins.py cube [nx ny nz]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF_SRC = os.environ.get("H2VIE_SRC", "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

from h2vie import arith, build, kernel  # noqa: E402
from h2vie.linalg import CompressionParams  # noqa: E402

from paper_1703_01175_b200.nearfield import assemble_near, geometry_arrays  # noqa: E402
from paper_1703_01175_b200.pack import pack_h2, save_packed, validate  # noqa: E402

K0 = 2.0 * np.pi
H = 1.0 / 16


def plane_wave_dirs(rng, count):
    """theta = arccos(U(-1, 1)), then phi = U(0, 2 pi), per wave."""
    out = []
    for _ in range(count):
        th = np.arccos(rng.uniform(-1, 1))
        ph = rng.uniform(0, 2 * np.pi)
        out.append([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])
    return np.asarray(out)


def build_op(dims, eps, n_min, tol):
    g = kernel.VoxelGeometry(kernel.lattice_centers(*dims, H), H ** 3, "pin")
    t = time.time()
    h2 = build.build_h2(g, kernel.KernelParams(K0, eps), CompressionParams(tol, tol), n_min=n_min,
                        eta=1.0)
    tb = time.time() - t
    pk = pack_h2(h2)
    validate(pk)
    print(f"built N={h2.n} in {tb:.0f} s; storage {h2.storage_bytes() / 1e6:.1f} MB, "
          f"far field {(pk.vbuf.nbytes + pk.tbuf.nbytes + pk.sbuf.nbytes) / 1e6:.1f} MB", flush=True)
    return g, h2, pk, tb


def geometry_record(dims, eps):
    rec = dict(kind="lattice", dims=list(dims), h=H, k0=K0)
    if np.ndim(eps) == 0:
        rec["eps_r"] = float(eps)
    else:
        rec["eps_r"] = {"uniform": [2.0, 6.0], "seed": 0}  # 2 + 4 * default_rng(0).random(N)
    return rec


def check_near(pk, geo):
    d = assemble_near(pk, *geometry_arrays(geo))
    err = np.max(np.abs(d - pk.dbuf)) / np.max(np.abs(pk.dbuf))
    print(f"re-assembled near-field max rel deviation {err:.2e}", flush=True)
    assert err < 1e-13


def make_plate(nx=256, ny=128):
    from oracle.krylov_oracle import gmres_solve
    dims = (nx, ny, 1)
    g, h2, pk, tb = build_op(dims, 4.0, 64, 1e-4)
    geo = geometry_record(dims, 4.0)
    check_near(pk, geo)
    d = plane_wave_dirs(np.random.default_rng(0), 1)[0]
    b = kernel.plane_wave_rhs(g, K0, d)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((h2.n, 2)) + 1j * rng.standard_normal((h2.n, 2))
    y = np.stack([arith.matvec(h2, x[:, 0]), arith.matvec(h2, x[:, 1])], 1)
    t = time.time()
    yb = arith.matvec(h2, b)
    tm = time.time() - t
    apply = lambda v: arith.matvec(h2, v)  # noqa: E731
    t = time.time()
    xs, rep = gmres_solve(apply, b, tol=1e-6, restart=50, max_iter=3000)
    tg = time.time() - t
    print(f"oracle GMRES(50): {rep.iterations} it, converged {rep.converged}, {tg:.0f} s", flush=True)
    extra = dict(x=x, y=y, rhs_plane_wave=b, y_plane_wave=yb, incidence=d, build_s=np.float64(tb),
                 ref_matvec_s=np.float64(tm), gmres_iters=np.int64(rep.iterations),
                 gmres_hist=np.asarray(rep.residual_history), gmres_x=xs, gmres_s=np.float64(tg))
    try:
        import scipy.sparse.linalg as sla
        cnt = [0]
        A = sla.LinearOperator((h2.n, h2.n), matvec=apply, dtype=np.complex128)
        sla.gmres(A, b, rtol=1e-6, atol=0.0, restart=50, maxiter=60,
                  callback=lambda _r: cnt.__setitem__(0, cnt[0] + 1), callback_type="pr_norm")
        extra["scipy_gmres_iters"] = np.int64(cnt[0])
        print(f"scipy GMRES(50): {cnt[0]} it", flush=True)
    except Exception as e:  # noqa: BLE001
        print("scipy cross-check skipped:", e)
    out = os.path.join(ROOT, "fixtures", f"pin_plate{nx}x{ny}.npz")
    save_packed(pk, out, extra=extra, geometry=geo)
    print(f"-> {out} {os.path.getsize(out) / 1e6:.1f} MB", flush=True)


def make_cube(nx=16, ny=16, nz=32, nrhs=64):
    from oracle.krylov_oracle import block_gmres_solve
    dims = (nx, ny, nz)
    n = nx * ny * nz
    eps = 2.0 + 4.0 * np.random.default_rng(0).random(n)
    g, h2, pk, tb = build_op(dims, eps, 64, 1e-4)
    geo = geometry_record(dims, eps)
    check_near(pk, geo)
    dirs = plane_wave_dirs(np.random.default_rng(0), nrhs)
    B = np.stack([kernel.plane_wave_rhs(g, K0, d) for d in dirs], 1)
    t = time.time()
    YB = arith.matmat_apply(h2, B)
    tm = time.time() - t
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, 1)) + 1j * rng.standard_normal((n, 1))
    y = arith.matvec(h2, x[:, 0])[:, None]
    t = time.time()
    Xs, rep = block_gmres_solve(lambda X: arith.matmat_apply(h2, X), B, tol=1e-6, restart=30,
                                max_iter=1000)
    tg = time.time() - t
    print(f"oracle block GMRES(30), {nrhs} RHS: {rep.iterations} block it, converged "
          f"{rep.converged}, {tg:.0f} s", flush=True)
    extra = dict(x=x, y=y, rhs_block=B, y_block=YB, dirs=dirs, build_s=np.float64(tb),
                 ref_matmat_s=np.float64(tm), bgmres_iters=np.int64(rep.iterations),
                 bgmres_hist=np.asarray(rep.residual_history), bgmres_x=Xs, bgmres_s=np.float64(tg))
    out = os.path.join(ROOT, "fixtures", f"pin_cube{nx}x{ny}x{nz}.npz")
    save_packed(pk, out, extra=extra, geometry=geo)
    print(f"-> {out} {os.path.getsize(out) / 1e6:.1f} MB", flush=True)


if __name__ == "__main__":
    kind = sys.argv[1]
    dims = [int(a) for a in sys.argv[2:]]
    if kind == "plate":
        make_plate(*dims)
    elif kind == "cube":
        make_cube(*dims)
    else:
        raise SystemExit(__doc__)
