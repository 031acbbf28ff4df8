"""The grouped complex GEMM / GEMV kernels behind every multi-RHS phase and every shard plan
(h2b_mrhs.cu: k_zgemm_grouped on DMMA for q >= 2, k_zgemv_grouped for q = 1), driven through
the plan C-ABI with random shapes — ragged m (1..64), k (1..32), row-major and transposed A,
accumulate and overwrite, every q-tile width — against the CPU interpreter of the same plan."""

import types

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _random_plan(rng, n_items, n_rows, q_rows):
    from paper_1703_01175_b200._abi import MM_ITEM, MM_SEG
    pays = [(rng.standard_normal(20000) + 1j * rng.standard_normal(20000)) for _ in range(6)]
    items, segs = [], []
    rows_used = 0
    for _ in range(n_items):
        m = int(rng.integers(1, 65))
        s0 = len(segs)
        trans = bool(rng.integers(0, 2))  # one A orientation per item (the GEMV kernel needs it)
        for _ in range(int(rng.integers(0, 6))):
            k = int(rng.integers(1, 33))
            lda = int(rng.integers(max(m, k) if trans else k, 70))
            if trans:
                lda = max(lda, m)
            else:
                lda = max(lda, k)
            span = (k - 1) * lda + m if trans else (m - 1) * lda + k
            a_off = int(rng.integers(0, 20000 - span))
            b_src = int(rng.integers(0, 3))
            b_row = int(rng.integers(0, q_rows - k))
            segs.append((a_off, b_row, k, lda, int(rng.integers(0, 6)) | (b_src << 4) | (256 if trans else 0), 0))
        acc = bool(rng.integers(0, 2))
        items.append((rows_used, m, s0, len(segs) - s0, 3 | (256 if acc else 0), 0))
        rows_used += m
    assert rows_used <= n_rows
    return pays, np.array(items, dtype=MM_ITEM), np.array(segs, dtype=MM_SEG)


@pytest.mark.parametrize("q", [1, 2, 7, 16, 33, 64, 100])
def test_grouped_kernels_match_interpreter(q):
    from oracle.plan_exec import NumpyPlanEngine
    from paper_1703_01175_b200.dist import CudaPlanEngine
    rng = np.random.default_rng(100 + q)
    n_rows, q_rows = 64 * 40, 600
    pays, items, segs = _random_plan(rng, 40, n_rows, q_rows)
    plan = types.SimpleNamespace(payloads=pays,
                                 phases={ph: (np.array([items.size], dtype=np.int64), items, segs)
                                         for ph in range(5)})
    X = rng.standard_normal((q_rows, q)) + 1j * rng.standard_normal((q_rows, q))
    YH = rng.standard_normal((q_rows, q)) + 1j * rng.standard_normal((q_rows, q))
    Y0 = rng.standard_normal((n_rows, q)) + 1j * rng.standard_normal((n_rows, q))
    ref = [torch.from_numpy(a.copy()) for a in (X, YH, Y0)]
    NumpyPlanEngine(plan).run(4, ref[0], ref[1], ref[2], q)
    eng = CudaPlanEngine(plan, 0)
    exp = ref[2].numpy()
    first = None
    for rep in range(5):  # repeated launches: a scheduling race shows up as a rare wrong tile
        dev = [torch.from_numpy(a.copy()).cuda() for a in (X, YH, Y0)]
        eng.run(4, dev[0], dev[1], dev[2], q)
        torch.cuda.synchronize()
        got = dev[2].cpu().numpy()
        assert np.linalg.norm(got - exp) <= 1e-13 * np.linalg.norm(exp), rep
        if first is None:
            first = got
        assert np.array_equal(got, first)  # deterministic: fixed summation order
    eng.close()


def test_plan_set_phase_validates_work_lists():
    """Malformed items/segments are rejected at upload (the kernels trust the lists)."""
    import ctypes as C
    from paper_1703_01175_b200 import _abi
    L = _abi.lib()
    h = C.c_void_p()
    elems = (C.c_int64 * 2)(4096, 4096)
    _abi.check(L.h2b_plan_create(0, 2, elems, C.byref(h)))

    def phase(items, segs, counts=None):
        it = np.array(items, dtype=_abi.MM_ITEM)
        sg = np.array(segs, dtype=_abi.MM_SEG)
        cnt = np.array(counts if counts is not None else [it.size], dtype=np.int64)
        return L.h2b_plan_set_phase(h, 0, int(cnt.size), cnt.ctypes.data_as(C.POINTER(C.c_int64)),
                                    it.ctypes.data, int(it.size), sg.ctypes.data, int(sg.size))

    ok_seg = (0, 0, 8, 8, 0, 0)
    assert phase([(0, 8, 0, 1, 3, 0)], [ok_seg]) == _abi.H2B_OK
    assert phase([(0, 65, 0, 1, 3, 0)], [ok_seg]) == _abi.H2B_EINVAL        # m > 64
    assert phase([(0, 8, 0, 2, 3, 0)], [ok_seg]) == _abi.H2B_EINVAL         # segments out of range
    assert phase([(0, 8, 0, 1, 3, 0)], [(0, 0, 33, 40, 0, 0)]) == _abi.H2B_EINVAL  # k > 32
    assert phase([(0, 8, 0, 1, 3, 0)], [(0, 0, 8, 8, 7, 0)]) == _abi.H2B_EINVAL    # no payload 7
    assert phase([(0, 8, 0, 2, 3, 0)], [ok_seg, (0, 0, 8, 8, 256, 0)]) == _abi.H2B_EINVAL  # mixed A
    assert phase([(0, 8, 0, 1, 3, 0)], [(0, 0, 8, 8, 512, 0)]) == _abi.H2B_EINVAL  # gather, no table
    assert phase([(0, 8, 0, 1, 3, 0)], [ok_seg], counts=[2]) == _abi.H2B_EINVAL     # counts mismatch
    _abi.check(L.h2b_plan_destroy(h))
