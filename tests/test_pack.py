"""Packed-format host logic (CPU only)."""

import numpy as np
import pytest

from conftest import GOLDEN_NAMES, load_golden
from paper_1703_01175_b200.pack import load_packed, save_packed, validate


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_validate_and_counts(name):
    pk, ex = load_golden(name)
    validate(pk)
    e = pk.element_counts()
    assert pk.storage_bytes() == pk.perm.nbytes + 16 * (e["E_V"] + e["E_T"] + e["E_S"] + e["E_D"])
    assert pk.algorithmic_bytes(1) == pk.storage_bytes() - pk.perm.nbytes + 32 * (pk.n + pk.total_rank)
    # children of a cluster are adjacent in their level (x̂_lo, x̂_hi contiguous)
    for p in range(pk.num_clusters):
        if pk.c_child_lo[p] >= 0:
            assert pk.c_child_hi[p] == pk.c_child_lo[p] + 1
            assert pk.c_parent[pk.c_child_lo[p]] == p
    # every leaf owns its diagonal near-field block (the near phase overwrites y)
    for p in pk.leaves():
        cols = pk.d_col[pk.d_row_ptr[p]:pk.d_row_ptr[p + 1]]
        assert p in cols


def test_roundtrip(tmp_path):
    pk, ex = load_golden("random137")
    path = tmp_path / "x.npz"
    save_packed(pk, path, extra={"y": ex["y"]})
    pk2, ex2 = load_packed(path, with_extra=True)
    for name in ("perm", "c_rank", "s_row_ptr", "d_off", "vbuf", "tbuf", "sbuf", "dbuf"):
        assert np.array_equal(getattr(pk, name), getattr(pk2, name))
    assert np.array_equal(ex2["y"], ex["y"])


def test_validate_rejects_broken_tiling():
    pk, _ = load_golden("rod164")
    import copy
    bad = copy.copy(pk)
    bad.d_row_ptr = pk.d_row_ptr.copy()
    bad.d_row_ptr[-1] -= 1
    bad.d_col = pk.d_col[:-1]
    with pytest.raises(ValueError):
        validate(bad)


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_payload_sizes_implied_by_tables(name):
    """E_V, E_T, E_S, E_D recomputed from the index tables equal the payload sizes (the sizes the
    device allocates for operators whose payloads are generated on the device)."""
    pk, _ = load_golden(name)
    assert pk.far_elems_expected() == (pk.vbuf.size, pk.tbuf.size, pk.sbuf.size)
    assert pk.d_elems_expected() == pk.dbuf.size


def test_structure_file_roundtrip(tmp_path):
    """save_structure keeps every table and the geometry; load_packed fills seeded payloads of the
    reference shapes (host) or leaves them for the device."""
    from paper_1703_01175_b200.pack import save_structure
    pk, _ = load_golden("cube8")
    geom = dict(kind="lattice", dims=[8, 8, 8], h=1 / 16, eps_r=4.0, k0=2 * np.pi)
    path = tmp_path / "s.npz"
    save_structure(pk, path, geom, seed=3)
    a = load_packed(path)
    b = load_packed(path)
    for t in ("c_start", "c_rank", "s_col", "s_off", "d_col", "d_off", "perm"):
        assert np.array_equal(getattr(a, t), getattr(pk, t))
    assert (a.vbuf.size, a.tbuf.size, a.sbuf.size) == (pk.vbuf.size, pk.tbuf.size, pk.sbuf.size)
    assert np.array_equal(a.sbuf, b.sbuf)                      # seeded: reproducible
    assert np.max(np.abs(a.dbuf - pk.dbuf)) <= 1e-14 * np.max(np.abs(pk.dbuf))  # near-field exact
    c = load_packed(path, near_on_host=False, far_on_host=False)
    assert c.sbuf.size == 0 and c.dbuf.size == 0 and "synthetic" in c.meta and "geometry" in c.meta
    assert c.algorithmic_bytes() == pk.algorithmic_bytes()


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_compact_structure_file_derives_offsets(name, tmp_path):
    """A compact structure file (compressed, without the payload offsets) loads to the same
    tables: the offsets are exactly the cumulative block sizes of the packer's order."""
    from paper_1703_01175_b200.pack import _INT_TABLES, save_structure
    pk, _ = load_golden(name)
    path = tmp_path / "c.npz"
    save_structure(pk, path, dict(kind="none"), seed=1, compact=True)
    assert "s_off" not in np.load(path).files
    c = load_packed(path, near_on_host=False, far_on_host=False)
    for t in _INT_TABLES:
        assert np.array_equal(getattr(c, t), getattr(pk, t)), t
