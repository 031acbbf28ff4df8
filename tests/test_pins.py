"""Reference-built pins of BASELINE configs 3 and 5 (tools/make_pins.py): CPU side.

* The right-hand sides follow SURVEY.md §8(d) exactly: a fresh default_rng(0), theta = arccos(U(-1, 1))
  then phi = U(0, 2 pi) per wave, e^{-j k0 d.r} at the voxel centres (kernel.py:237-242).  The
  product's plane_wave_rhs / seeded_incidence regenerate the reference's stored vectors bit for bit.
* The oracle restatement of arith.matvec reproduces the reference's own outputs stored in the pins.
"""

import os

import numpy as np
import pytest

from conftest import ROOT, rel

PLATE = os.path.join(ROOT, "fixtures", "pin_plate256x128.npz")
CUBE = os.path.join(ROOT, "fixtures", "pin_cube16x16x32.npz")


def _load(path, **kw):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not present (tools/make_pins.py)")
    from paper_1703_01175_b200.pack import load_packed
    return load_packed(path, with_extra=True, **kw)


def test_plate_plane_wave_rhs_is_the_reference_one():
    from paper_1703_01175_b200.nearfield import geometry_arrays, plane_wave_rhs, seeded_incidence
    pk, ex = _load(PLATE, near_on_host=False)
    centers, _, k0, _ = geometry_arrays(pk.meta["geometry"])
    d = seeded_incidence(np.random.default_rng(0))
    assert np.array_equal(d, ex["incidence"])
    assert np.array_equal(plane_wave_rhs(centers, k0, d), ex["rhs_plane_wave"])
    # the oracle GMRES(50) count on it is scipy's too (the reference has no GMRES)
    assert int(ex["gmres_iters"]) == int(ex["scipy_gmres_iters"])


def test_cube_plane_waves_are_the_reference_ones():
    from paper_1703_01175_b200.nearfield import geometry_arrays, plane_wave_rhs, seeded_incidence
    pk, ex = _load(CUBE, near_on_host=False)
    centers, chi, k0, _ = geometry_arrays(pk.meta["geometry"])
    rng = np.random.default_rng(0)
    dirs = np.stack([seeded_incidence(rng) for _ in range(64)])
    assert np.array_equal(dirs, ex["dirs"])
    B = np.stack([plane_wave_rhs(centers, k0, d) for d in dirs], 1)
    assert np.array_equal(B, ex["rhs_block"])
    # eps_r = 2 + 4 U[0, 1) per cell from default_rng(0) (SURVEY.md §8d cfg 5)
    assert np.allclose(chi + 1.0, 2.0 + 4.0 * np.random.default_rng(0).random(pk.n), rtol=0, atol=0)


@pytest.mark.parametrize("path", [CUBE, PLATE])
def test_oracle_matches_reference_on_pins(path):
    from oracle import h2_oracle as ho
    pk, ex = _load(path)
    assert rel(ho.matvec(pk, ex["x"][:, 0]), ex["y"][:, 0]) <= 1e-12
