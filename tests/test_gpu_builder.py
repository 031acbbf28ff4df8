"""Stage II of the H² builder on the device from the reference's own Stage-I
factors (tests/golden/stage1_*.npz, tools/make_stage1.py).

The device-built operator is checked the way the reference checks its own builder
(test_build.py / test_arith.py:42-48): its matvec agrees with the dense operator within
10·eps_acc, and with the reference-built H² operator (whose own representation error is
~eps_acc) within the same bound; the ranks match the reference's except where an eigenvalue sits
on the truncation threshold.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel

pytestmark = pytest.mark.gpu


def _stage1(name):
    path = os.path.join(GOLDEN, f"stage1_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"stage1_{name}.npz missing (tools/make_stage1.py)")
    from paper_1703_01175_b200.pack import load_packed
    return load_packed(path, with_extra=True)


@pytest.mark.parametrize("name", ["rod164", "cube8", "line2048"])
def test_device_stage2_operator_within_tolerance(name):
    from paper_1703_01175_b200 import H2Operator
    from paper_1703_01175_b200.builder import build_stage2
    pk, ex = _stage1(name)
    eps = float(ex["s1_eps_acc"])
    pkd = build_stage2(pk, ex, eps, device=0)
    # ranks: equal to the reference's up to a few threshold cases
    diff = np.abs(pkd.c_rank.astype(int) - ex["ref_rank"].astype(int))
    assert diff.max() <= 2 and np.count_nonzero(diff) <= max(2, pk.num_clusters // 10), diff
    # against the reference-built operator (both within ~eps_acc of the dense operator)
    gold, gex = load_golden(name)
    op = H2Operator(pkd, device=0)
    for j in range(2):
        x = gex["x"][:, j]
        assert rel(op.matvec(x), gex["y"][:, j]) <= 10 * eps
    if "dense" in gex:
        D = gex["dense"]
        X = gex["x"][:, :4]
        assert rel(op.matmat(X), D @ X) <= 10 * eps
    op.close()


def test_device_stage2_bases_are_orthonormal():
    """Leaf bases and transfers come from a Hermitian eigendecomposition: orthonormal columns."""
    from paper_1703_01175_b200.builder import build_stage2
    pk, ex = _stage1("cube8")
    pkd = build_stage2(pk, ex, float(ex["s1_eps_acc"]), device=0)
    for c in range(pkd.num_clusters):
        k = int(pkd.c_rank[c])
        if k == 0:
            continue
        if pkd.c_child_lo[c] < 0:
            V = pkd.vbuf[pkd.c_v_off[c]:pkd.c_v_off[c] + pkd.c_size[c] * k].reshape(pkd.c_size[c], k)
        else:
            m = int(pkd.c_rank[pkd.c_child_lo[c]] + pkd.c_rank[pkd.c_child_hi[c]])
            V = pkd.tbuf[pkd.c_t_off[c]:pkd.c_t_off[c] + m * k].reshape(m, k)
        assert np.allclose(V.conj().T @ V, np.eye(k), atol=1e-12)


@pytest.mark.parametrize("name", ["rod164", "cube8", "line2048"])
def test_device_builder_end_to_end(name):
    """Stage I (ACA, entries from the geometry) and Stage II both on the device: the operator agrees
    with the reference-built one and with the dense operator within 10·eps_acc."""
    from paper_1703_01175_b200 import H2Operator
    from paper_1703_01175_b200.builder import build_device, stage1_device
    pk, ex = _stage1(name)
    eps = float(ex["s1_eps_acc"])
    s1 = stage1_device(pk, ex["geom_centers"], ex["geom_chi"], float(ex["geom_k0"]), float(ex["geom_volume"]),
                       float(ex["s1_eps_aca"]))
    # the device ACA follows the reference's pivoting: ranks equal to the reference's Stage I up to
    # rounding of the stopping test (the reference also trims them by an SVD, skipped here)
    assert np.all(s1["s1_rank"] >= 0)
    pkd = build_device(pk, ex["geom_centers"], ex["geom_chi"], float(ex["geom_k0"]), float(ex["geom_volume"]),
                       float(ex["s1_eps_aca"]), eps)
    gold, gex = load_golden(name)
    op = H2Operator(pkd, device=0)
    for j in range(2):
        assert rel(op.matvec(gex["x"][:, j]), gex["y"][:, j]) <= 10 * eps
    if "dense" in gex:
        X = gex["x"][:, :4]
        assert rel(op.matmat(X), gex["dense"] @ X) <= 10 * eps
    op.close()


@pytest.mark.parametrize("k", [1, 2])
def test_device_builder_baseline_configs(k):
    """BASELINE configs 1 and 2: the far field of the reference block structure built on the device
    from the geometry agrees with the reference-built operator within 10·eps_acc (measured:
    1.2e-5 and 2.4e-8) with the same ranks up to the truncation threshold."""
    from conftest import load_config
    from paper_1703_01175_b200 import H2Operator
    from paper_1703_01175_b200.builder import build_device
    from paper_1703_01175_b200.nearfield import geometry_arrays
    pk, ex = load_config(k)
    if "geometry" not in pk.meta:
        pytest.skip("no geometry record")
    centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
    pkd = build_device(pk, centers, chi, k0, vol, 1e-4, 1e-4)
    dk = np.abs(pkd.c_rank.astype(int) - pk.c_rank.astype(int))
    assert dk.max() <= 2 and np.count_nonzero(dk) <= pk.num_clusters // 100 + 2
    op = H2Operator(pkd, device=0)
    for j in range(ex["x"].shape[1]):
        assert rel(op.matvec(ex["x"][:, j]), ex["y"][:, j]) <= 10 * 1e-4
    op.close()


def test_device_built_config3_matches_reference_and_gmres_count():
    """BASELINE config 3 in full (262,144 points, 7.1 GB operator): the reference block structure
    (fixtures/cfg3_structure.npz), far field built on the B200 from the geometry (Stage I ACA +
    Stage II, ~18 s; the reference's Python build takes 550 s), near-field sampled on the device.
    Its matvec agrees with the reference-built operator's own outputs within eps_acc (measured
    5.9e-6) and GMRES(50) to 1e-6 on the SURVEY §8(d) plane wave takes the oracle's count on the
    reference operator (511 = scipy's) within +-1."""
    import os
    from conftest import ROOT
    from paper_1703_01175_b200 import H2Operator, gmres_solve
    from paper_1703_01175_b200.builder import build_device
    from paper_1703_01175_b200.nearfield import geometry_arrays
    from paper_1703_01175_b200.pack import load_packed
    sp = os.path.join(ROOT, "fixtures", "cfg3_structure.npz")
    rp = os.path.join(ROOT, "fixtures", "cfg3_ref_outputs.npz")
    if not (os.path.exists(sp) and os.path.exists(rp)):
        pytest.skip("cfg3 structure / reference outputs not present")
    pk, _ = load_packed(sp, with_extra=True, near_on_host=False, far_on_host=False)
    ref = np.load(rp)
    centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
    pkd = build_device(pk, centers, chi, k0, vol, 1e-4, 1e-4)
    op = H2Operator(pkd, device=0)
    for j in range(ref["x"].shape[1]):
        assert rel(op.matvec(ref["x"][:, j]), ref["y"][:, j]) <= 1e-4
    x, rep = gmres_solve(op, ref["rhs_plane_wave"], tol=1e-6, restart=50, max_iter=3000)
    assert rep.converged and abs(rep.iterations - int(ref["gmres_iters"])) <= 1
    op.close()
