"""The C-ABI library loads and exports every symbol include/h2b.h declares (CPU only)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "h2b.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(h2b_\w+)\s*\(", src, re.M)))


def test_header_declares_the_surface():
    names = _declared()
    for must in ("h2b_create", "h2b_upload", "h2b_matvec_perm", "h2b_matvec_host", "h2b_gmres",
                 "h2b_bicgstab", "h2b_destroy", "h2b_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1703_01175_b200 import _abi
    L = _abi.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_abi.EXPORTED) == set(_declared())
    assert L.h2b_version() == 1


def test_library_is_sm100a_only():
    """The .so carries sm_100a SASS (no PTX/JIT or other-arch fallback)."""
    import subprocess
    from paper_1703_01175_b200 import _abi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_no_device_means_loud_failure():
    """Without a B200 the product path raises instead of falling back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1703_01175_b200 import H2Operator, _abi
    assert _abi.lib().h2b_device_ok(0) == 0
    pk, _ = load_golden("rod164")
    with pytest.raises(RuntimeError):
        H2Operator(pk)
    from paper_1703_01175_b200 import matvec
    with pytest.raises(RuntimeError):
        matvec(pk, np.zeros(pk.n))


def test_create_rejects_without_device_with_status():
    import ctypes as C
    from paper_1703_01175_b200 import _abi
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lay = _abi.Layout()
    h = C.c_void_p()
    rc = _abi.lib().h2b_create(C.byref(lay), 0, C.byref(h))
    assert rc == _abi.H2B_ENODEV
    assert b"no CPU fallback" in _abi.lib().h2b_last_error()


def test_plan_create_without_device_fails_loudly():
    import ctypes as C
    import torch
    from paper_1703_01175_b200 import _abi
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    elems = (C.c_int64 * 1)(4)
    assert _abi.lib().h2b_plan_create(0, 1, elems, C.byref(h)) == _abi.H2B_ENODEV
