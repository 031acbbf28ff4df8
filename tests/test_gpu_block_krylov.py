"""Block GMRES(m) on device vs the CPU restatement (oracle/krylov_oracle.py::block_gmres_solve)."""

import numpy as np
import pytest

from conftest import load_config, load_golden, rel

pytestmark = pytest.mark.gpu


def _seeded_rhs(pk, q, seed):
    """q seeded complex N(0,1) right-hand sides (the plane-wave block of cfg5 is in test_gpu_pins.py)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((pk.n, q)) + 1j * rng.standard_normal((pk.n, q))


@pytest.mark.parametrize("name,q,m", [("rod164", 4, 10), ("cube8", 3, 8), ("plate32", 5, 6),
                                      ("random137", 2, 5)])
def test_block_gmres_matches_oracle(name, q, m):
    from oracle import h2_oracle as ho
    from oracle import krylov_oracle as ko
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve
    pk, _ = load_golden(name)
    B = _seeded_rhs(pk, q, 3)
    op = H2Operator(pk)
    X, rep = block_gmres_solve(op, B, tol=1e-8, restart=m, max_iter=400)
    Xo, ro = ko.block_gmres_solve(lambda V: ho.matmat_apply(pk, V), B, tol=1e-8, restart=m, max_iter=400)
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 1, (rep.iterations, ro.iterations)
    res = np.linalg.norm(ho.matmat_apply(pk, X) - B, axis=0) / np.linalg.norm(B, axis=0)
    assert res.max() <= 1e-8
    assert rel(X, Xo) <= 1e-6
    op.close()


def test_block_gmres_single_column_equals_gmres():
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve, gmres_solve
    pk, ex = load_golden("rod164")
    op = H2Operator(pk)
    b = ex["x"][:, 0]
    xb, rb = block_gmres_solve(op, b[:, None], tol=1e-8, restart=20, max_iter=300)
    xg, rg = gmres_solve(op, b, tol=1e-8, restart=20, max_iter=300)
    assert abs(rb.iterations - rg.iterations) <= 1
    assert rel(xb[:, 0], xg) <= 1e-6
    op.close()


def test_block_gmres_cfg1_q8():
    from oracle import h2_oracle as ho
    from oracle import krylov_oracle as ko
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve
    pk, ex = load_config(1)
    B = _seeded_rhs(pk, 8, 11)
    B[:, 0] = ex["x"][:, 0]
    op = H2Operator(pk)
    X, rep = block_gmres_solve(op, B, tol=1e-6, restart=30, max_iter=600)
    Xo, ro = ko.block_gmres_solve(lambda V: ho.matmat_apply(pk, V), B, tol=1e-6, restart=30, max_iter=600)
    assert rep.converged and abs(rep.iterations - ro.iterations) <= 1, (rep.iterations, ro.iterations)
    res = np.linalg.norm(ho.matmat_apply(pk, X) - B, axis=0) / np.linalg.norm(B, axis=0)
    assert res.max() <= 1e-6
    op.close()


def test_block_gmres_zero_rhs_and_argument_checks():
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve
    pk, _ = load_golden("rod164")
    op = H2Operator(pk)
    X, rep = block_gmres_solve(op, np.zeros((pk.n, 3)))
    assert rep.converged and rep.iterations == 0 and not X.any()
    with pytest.raises(ValueError):
        block_gmres_solve(op, np.zeros(pk.n))
    with pytest.raises(ValueError):
        block_gmres_solve(op, np.ones((pk.n, 2)), tol=1.5)
    op.close()


def test_block_gmres_history_follows_oracle():
    """The per-step residual history (max over columns of the least-squares residual) follows the
    oracle's."""
    from oracle import h2_oracle as ho
    from oracle import krylov_oracle as ko
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve
    pk, _ = load_golden("rod164")
    B = _seeded_rhs(pk, 4, 5)
    op = H2Operator(pk)
    X, rep = block_gmres_solve(op, B, tol=1e-8, restart=10, max_iter=400)
    Xo, ro = ko.block_gmres_solve(lambda V: ho.matmat_apply(pk, V), B, tol=1e-8, restart=10, max_iter=400)
    assert rep.converged and abs(rep.iterations - ro.iterations) <= 1
    k = min(8, len(rep.residual_history), len(ro.residual_history))
    assert np.allclose(rep.residual_history[:k], ro.residual_history[:k], rtol=1e-5)
    op.close()


def test_block_gmres_zero_column():
    """An all-zero right-hand side column (norm taken as 1, as in the oracle) deflates: its
    solution column is exactly zero and the other columns converge as usual.  (The oracle's
    Householder QR fills the deflated basis column with an arbitrary orthonormal direction, so
    its Krylov space, and its iteration count, may differ slightly.)"""
    from oracle import h2_oracle as ho
    from paper_1703_01175_b200 import H2Operator, block_gmres_solve
    pk, _ = load_golden("rod164")
    B = _seeded_rhs(pk, 4, 5)
    B[:, 2] = 0.0
    op = H2Operator(pk)
    X, rep = block_gmres_solve(op, B, tol=1e-8, restart=10, max_iter=400)
    assert rep.converged and not np.any(X[:, 2])
    res = np.linalg.norm(ho.matmat_apply(pk, X) - B, axis=0) / np.where(np.linalg.norm(B, axis=0) == 0, 1,
                                                                        np.linalg.norm(B, axis=0))
    assert res.max() <= 1e-8
    op.close()
