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
