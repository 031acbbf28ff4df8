"""Pin the CPU oracle against vectors produced by the reference itself (CPU only)."""

import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_config, load_golden, rel
from oracle import h2_oracle as ho
from oracle import krylov_oracle as ko


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_partition_bit_exact(name):
    pk, ex = load_golden(name)
    assert np.array_equal(pk.perm, ex["ref_perm"])
    assert pk.admissible_pairs() == [tuple(r) for r in ex["ref_admissible"].tolist()]
    assert pk.inadmissible_pairs() == [tuple(r) for r in ex["ref_inadmissible"].tolist()]
    assert int(ex["ref_tiling"]) == pk.n * pk.n
    assert pk.storage_bytes() == int(ex["ref_storage_bytes"])


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_loop_oracle_matches_reference_matvec(name):
    pk, ex = load_golden(name)
    for j in range(ex["x"].shape[1]):
        assert rel(ho.matvec(pk, ex["x"][:, j]), ex["y"][:, j]) <= 1e-13


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_packed_oracle_matches_reference_matvec(name):
    pk, ex = load_golden(name)
    xp = ex["x"][pk.perm]
    yp = ho.matvec_perm_packed(pk, xp)
    y = np.empty_like(yp)
    y[pk.perm] = yp
    assert rel(y, ex["y"]) <= 1e-13


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_oracle_matmat_and_chunking(name):
    pk, ex = load_golden(name)
    assert rel(ho.matmat_apply(pk, ex["xm"]), ex["ym"]) <= 1e-13
    assert rel(ho.matmat_apply(pk, ex["xm"], col_block=2), ex["ym_cb2"]) <= 1e-13


def test_oracle_exact_cases():
    pk, ex = load_golden("rod164")
    assert np.array_equal(ho.matvec(pk, np.zeros(pk.n)), np.zeros(pk.n))
    pk, ex = load_golden("identity")
    x = ex["x"][:, 0]
    assert np.array_equal(ho.matvec(pk, x), x)
    assert np.array_equal(ex["y"][:, 0], x)  # the reference agrees (test_arith.py:37-40)


@pytest.mark.parametrize("name", ["rod164", "cube2"])
def test_oracle_within_compression_tolerance_of_dense(name):
    pk, ex = load_golden(name)
    for j in range(ex["x"].shape[1]):
        ref = ex["dense"] @ ex["x"][:, j]
        assert rel(ho.matvec(pk, ex["x"][:, j]), ref) <= 10 * pk.meta["eps_acc"]


def test_oracle_rejects_wrong_length():
    pk, _ = load_golden("rod164")
    with pytest.raises(ValueError):
        ho.matvec(pk, np.zeros(pk.n + 1))
    with pytest.raises(ValueError):
        ho.matmat_apply(pk, np.zeros(pk.n))


@pytest.mark.parametrize("name", ["rod164", "cube2"])
@pytest.mark.parametrize("tag", ["e3", "e6"])
def test_bicgstab_oracle_matches_reference(name, tag):
    pk, ex = load_golden(name)
    x, rep = ko.bicgstab_solve(lambda v: ho.matvec(pk, v), ex["bicg_rhs"],
                               tol={"e3": 1e-3, "e6": 1e-6}[tag], max_iter=400)
    assert rep.iterations == int(ex[f"bicg_{tag}_iters"])
    assert rep.converged == bool(ex[f"bicg_{tag}_conv"])
    assert np.allclose(rep.residual_history, ex[f"bicg_{tag}_hist"], rtol=1e-6, atol=0)
    assert rel(x, ex[f"bicg_{tag}_x"]) <= 1e-8


def test_bicgstab_oracle_edge_cases(rng):
    b = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    x, rep = ko.bicgstab_solve(lambda v: v, b, tol=1e-10)
    assert rep.converged and rep.iterations <= 1 and np.allclose(x, b)
    x, rep = ko.bicgstab_solve(lambda v: v, np.zeros(10), tol=1e-3)
    assert rep.iterations == 0 and rep.converged
    with pytest.raises(ValueError):
        ko.bicgstab_solve(lambda v: v, np.ones(4), tol=0.0)
    with pytest.raises(ValueError):
        ko.bicgstab_solve(lambda v: v, np.ones(4), tol=1e-3, max_iter=0)


@pytest.mark.parametrize("name,restart", [("rod164", 30), ("cube2", 10), ("plate32", 20),
                                          ("line2048", 30)])
def test_gmres_oracle_matches_scipy_iterations(name, restart):
    scipy_la = pytest.importorskip("scipy.sparse.linalg")
    pk, ex = load_golden(name)
    b = ex["x"][:, 0]
    x, rep = ko.gmres_solve(lambda v: ho.matvec_perm_packed(pk, v[pk.perm])[np.argsort(pk.perm)],
                            b, tol=1e-8, restart=restart, max_iter=2000)
    assert rep.converged
    A = scipy_la.LinearOperator((pk.n, pk.n), dtype=np.complex128,
                                matvec=lambda v: ho.matvec_perm_packed(pk, v[pk.perm])[np.argsort(pk.perm)])
    count = [0]
    xs, info = scipy_la.gmres(A, b, rtol=1e-8, atol=0, restart=restart, maxiter=2000,
                              callback=lambda r: count.__setitem__(0, count[0] + 1),
                              callback_type="pr_norm")
    assert info == 0
    assert abs(rep.iterations - count[0]) <= 1
    assert rel(x, xs) <= 1e-6


def test_gmres_oracle_edge_cases(rng):
    b = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    x, rep = ko.gmres_solve(lambda v: v, b, tol=1e-10, restart=5)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b)
    x, rep = ko.gmres_solve(lambda v: v, np.zeros(7), tol=1e-3)
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    with pytest.raises(ValueError):
        ko.gmres_solve(lambda v: v, b, tol=1.5)


def test_block_gmres_oracle_solves(rng):
    pk, ex = load_golden("cube2")
    B = ex["xm"][:, :3]
    ap = lambda X: ho.matmat_apply(pk, X)
    X, rep = ko.block_gmres_solve(ap, B, tol=1e-8, restart=10)
    assert rep.converged
    assert np.linalg.norm(ap(X) - B, axis=0).max() / np.linalg.norm(B, axis=0).min() <= 1e-7


def test_config1_reference_outputs_and_gmres_count():
    pk, ex = load_config(1)
    assert np.array_equal(pk.perm, ex["ref_perm"])
    assert int(ex["ref_tiling"]) == pk.n ** 2
    assert rel(ho.matvec_perm_packed(pk, ex["x"][pk.perm, 0]), ex["y"][pk.perm, 0]) <= 1e-13
    # SURVEY.md §0 finding 1: GMRES(30) to 1e-6 takes 245 iterations on config 1
    assert abs(int(ex["gmres_iters"]) - 245) <= 1


def test_config2_reference_outputs():
    pk, ex = load_config(2)
    assert np.array_equal(pk.perm, ex["ref_perm"])
    assert abs(pk.algorithmic_bytes() / 1e6 - 121.8) < 0.1
    assert rel(ho.matvec_perm_packed(pk, ex["x"][pk.perm, 0]), ex["y"][pk.perm, 0]) <= 1e-13
