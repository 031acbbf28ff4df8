"""GPU parity on the reference-built pins of BASELINE configs 3 and 5 (tools/make_pins.py).

* plate (cfg3 construction: 16 points/lambda, eps_r 4, leaf 64, tol 1e-4; 256 x 128 points, the
  largest plate whose compact file ships to the GPU box): matvec <= 1e-10 against the reference's
  own arith.matvec outputs; GMRES(50) to 1e-6 on the SURVEY §8(d) plane wave with the oracle's
  iteration count +-1 (= scipy's).
* cube (cfg5 construction: random eps_r in [2, 6] per cell, leaf 64, tol 1e-4; 16 x 16 x 32
  points): matvec and the 64-plane-wave matmat_apply <= 1e-10 against the reference; block
  GMRES(30) over the 64 plane waves to 1e-6 with the oracle's block-iteration count +-1.
"""

import os

import numpy as np
import pytest

from conftest import ROOT, rel

pytestmark = pytest.mark.gpu

PLATE = os.path.join(ROOT, "fixtures", "pin_plate256x128.npz")
CUBE = os.path.join(ROOT, "fixtures", "pin_cube16x16x32.npz")
_ops = {}


def _op(path):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not present (tools/make_pins.py)")
    if path not in _ops:
        from paper_1703_01175_b200 import H2Operator
        from paper_1703_01175_b200.pack import load_packed
        pk, ex = load_packed(path, with_extra=True, near_on_host=False)  # near-field sampled in HBM
        _ops[path] = (H2Operator(pk, device=0), pk, ex)
    return _ops[path]


@pytest.mark.parametrize("path", [PLATE, CUBE])
def test_pin_matvec_matches_reference(path):
    op, pk, ex = _op(path)
    for j in range(ex["x"].shape[1]):
        assert rel(op.matvec(ex["x"][:, j]), ex["y"][:, j]) <= 1e-10
    if "y_plane_wave" in ex:
        assert rel(op.matvec(ex["rhs_plane_wave"]), ex["y_plane_wave"]) <= 1e-10


def test_pin_cube_matmat_matches_reference():
    from paper_1703_01175_b200 import matmat_apply
    op, pk, ex = _op(CUBE)
    Y = matmat_apply(op, ex["rhs_block"])
    assert rel(Y, ex["y_block"]) <= 1e-10
    for j in (0, 17, 63):
        assert rel(Y[:, j], ex["y_block"][:, j]) <= 1e-10


def test_pin_plate_gmres50_iterations_match_oracle():
    from paper_1703_01175_b200 import gmres_solve
    op, pk, ex = _op(PLATE)
    b = ex["rhs_plane_wave"]
    x, rep = gmres_solve(op, b, tol=1e-6, restart=50, max_iter=3000)
    assert rep.converged
    assert abs(rep.iterations - int(ex["gmres_iters"])) <= 1
    assert rel(x, ex["gmres_x"]) <= 1e-5
    assert np.linalg.norm(op.matvec(x) - b) / np.linalg.norm(b) <= 1e-6
    k = min(20, len(rep.residual_history))
    assert np.allclose(rep.residual_history[:k], ex["gmres_hist"][:k], rtol=1e-6)


def test_pin_cube_block_gmres_iterations_match_oracle():
    from paper_1703_01175_b200 import block_gmres_solve
    op, pk, ex = _op(CUBE)
    B = ex["rhs_block"]
    X, rep = block_gmres_solve(op, B, tol=1e-6, restart=30, max_iter=1000)
    assert rep.converged
    assert abs(rep.iterations - int(ex["bgmres_iters"])) <= 1
    R = op.matmat(X) - B
    assert np.max(np.linalg.norm(R, axis=0) / np.linalg.norm(B, axis=0)) <= 1e-6
    assert rel(X, ex["bgmres_x"]) <= 1e-5
