"""Build the far field of a BASELINE operator (cfg1 / cfg2 / cfg3 / cfg5)'s block structure on the B200 (Stage I ACA + Stage II)
from the voxel geometry, and compare its matvec with the reference-built operator's stored
outputs.  Usage: python tools/build_device.py cfg2 [cfg1 ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_01175_b200 import H2Operator  # noqa: E402
from paper_1703_01175_b200.builder import build_stage2, stage1_device  # noqa: E402
from paper_1703_01175_b200.nearfield import geometry_arrays  # noqa: E402
from paper_1703_01175_b200.pack import load_packed  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    if name == "cfg3":  # the reference block structure + the reference's own matvec outputs
        pk, _ = load_packed(os.path.join(ROOT, "fixtures", "cfg3_structure.npz"), with_extra=True,
                            near_on_host=False, far_on_host=False)
        ex = dict(np.load(os.path.join(ROOT, "fixtures", "cfg3_ref_outputs.npz")))
    elif name in ("cfg4", "cfg5"):  # reference block structure, no reference outputs (cannot be built here)
        pk, _ = load_packed(os.path.join(ROOT, "fixtures", f"{name}_structure.npz"), with_extra=True,
                            near_on_host=False, far_on_host=False)
        ex = {}
    else:
        pk, ex = load_packed(os.path.join(ROOT, "fixtures", name + ".npz"), with_extra=True, near_on_host=False)
    centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
    eps = float(pk.meta.get("eps_acc", 1e-4)) or 1e-4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s1 = stage1_device(pk, centers, chi, k0, vol, eps)
    t1 = time.perf_counter()
    pkd = build_stage2(pk, s1, eps)
    t2 = time.perf_counter()
    op = H2Operator(pkd, device=0)
    errs = [float(np.linalg.norm(op.matvec(ex["x"][:, j]) - ex["y"][:, j]) / np.linalg.norm(ex["y"][:, j]))
            for j in range(ex["x"].shape[1])] if "x" in ex else [float("nan")]
    dk = np.abs(pkd.c_rank.astype(int) - pk.c_rank.astype(int))
    gm = ""
    # sampled rows against the exact operator (direct sums over all N columns on the device)
    from paper_1703_01175_b200.builder import exact_rows
    rng = np.random.default_rng(3)
    xr = rng.standard_normal(pk.n) + 1j * rng.standard_normal(pk.n)
    rows = np.sort(rng.choice(pk.n, 256, replace=False))
    ye = exact_rows(rows, xr, centers, chi, k0, vol)
    yh = op.matvec(xr)[rows]
    gm += f"; 256 sampled rows vs the exact operator: {np.linalg.norm(yh - ye) / np.linalg.norm(ye):.2e}"
    if name == "cfg5":  # 64 plane waves, block GMRES(30) to 1e-6
        from paper_1703_01175_b200 import block_gmres_solve
        from paper_1703_01175_b200.nearfield import plane_wave_rhs, seeded_incidence
        rng0 = np.random.default_rng(0)
        Bw = np.stack([plane_wave_rhs(centers, k0, seeded_incidence(rng0)) for _ in range(64)], 1)
        Xw, rep = block_gmres_solve(op, Bw, tol=1e-6, restart=30, max_iter=1000)
        res = np.linalg.norm(op.matmat(Xw) - Bw, axis=0) / np.linalg.norm(Bw, axis=0)
        gm += (f"; block GMRES(30), 64 plane waves, to 1e-6: {rep.iterations} block it, {rep.wall_time:.2f} s, "
               f"converged {rep.converged}, max true residual {res.max():.2e}")
    if "rhs_plane_wave" in ex:  # GMRES(50) on the BASELINE cfg3 plane wave (SURVEY 8d draw)
        from paper_1703_01175_b200 import gmres_solve
        xg, rep = gmres_solve(op, ex["rhs_plane_wave"], tol=1e-6, restart=50, max_iter=3000)
        gm += (f"; GMRES(50) to 1e-6: {rep.iterations} it (reference operator, oracle: "
              f"{int(ex['gmres_iters'])}), {rep.wall_time:.3f} s, converged {rep.converged}")
    print(f"{name}: N={pk.n} Stage I {t1 - t0:.2f} s (ACA ranks max {int(s1['s1_rank'].max())}), Stage II "
          f"{t2 - t1:.2f} s; ranks vs reference: {int(np.count_nonzero(dk))} of {pk.num_clusters} differ "
          f"(max {int(dk.max())}); K {int(pkd.c_rank.sum())} vs {int(pk.c_rank.sum())}; matvec vs the "
          f"reference-built operator {max(errs):.2e} (eps_acc {eps:g})" + gm, flush=True)
    op.close()
