"""Near-field re-assembly from geometry (nearfield.py) vs the reference-built payloads."""

import os

import numpy as np
import pytest

from conftest import ROOT, load_golden, rel
from paper_1703_01175_b200.nearfield import assemble_near, geometry_arrays
from paper_1703_01175_b200.pack import load_packed

TWO_PI = 2 * np.pi
LATTICE = {  # tools/make_golden.py make_small(): scaled BASELINE shapes
    "cube8": dict(kind="lattice", dims=[8, 8, 8], h=1 / 16, eps_r=4.0, k0=TWO_PI),
    "line2048": dict(kind="lattice", dims=[2048, 1, 1], h=1 / 32, eps_r=4.0, k0=TWO_PI),
    "plate32": dict(kind="lattice", dims=[32, 32, 1], h=1 / 16, eps_r=4.0, k0=TWO_PI),
}


@pytest.mark.parametrize("name", sorted(LATTICE))
def test_reassembled_near_field_matches_reference(name):
    pk, _ = load_golden(name)
    d = assemble_near(pk, *geometry_arrays(LATTICE[name]))
    assert d.shape == pk.dbuf.shape
    assert np.max(np.abs(d - pk.dbuf)) <= 1e-14 * np.max(np.abs(pk.dbuf))


@pytest.mark.parametrize("k", [1, 2])
def test_compact_fixture_reproduces_reference_matvec(k):
    """fixtures/cfg<k>.npz (no near-field payload) -> oracle matvec == reference arith.matvec."""
    from oracle import h2_oracle as ho
    path = os.path.join(ROOT, "fixtures", f"cfg{k}.npz")
    pk, ex = load_packed(path, with_extra=True)
    assert pk.dbuf.size == pk.d_elems_expected() > 0
    y = ho.matvec(pk, ex["x"][:, 0])
    assert rel(y, ex["y"][:, 0]) <= 1e-12
    full = os.path.join(ROOT, "data", f"cfg{k}.npz")
    if os.path.exists(full):
        assert np.array_equal(load_packed(full).dbuf, pk.dbuf)


@pytest.mark.parametrize("name", ["cube8", "line2048", "plate32"])
def test_plane_wave_rhs_matches_reference(name):
    """plane_wave_rhs restates kernel.plane_wave_rhs (kernel.py:237-242): bit-identical to the
    right-hand side the reference generated for the golden BiCGStab solves."""
    from paper_1703_01175_b200.nearfield import plane_wave_rhs
    _, ex = load_golden(name)
    centers, _, k0, _ = geometry_arrays(LATTICE[name])
    assert np.array_equal(plane_wave_rhs(centers, k0, [0, -1, 0]), ex["bicg_rhs"])
    with pytest.raises(ValueError):
        plane_wave_rhs(centers, k0, [1, 1, 0])
