"""Shared fixtures.  GPU tests are marked `gpu`; everything else runs on CPU."""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")

GOLDEN_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                      if not os.path.basename(p).startswith("stage1_"))  # Stage-I factors: builder tests


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: takes more than ~20 s on CPU")


_cache = {}


def load_golden(name):
    """(PackedH2, extras) for tests/golden/<name>.npz — outputs of the reference itself."""
    if name not in _cache:
        from paper_1703_01175_b200.pack import load_packed
        _cache[name] = load_packed(os.path.join(GOLDEN, name + ".npz"), with_extra=True)
    return _cache[name]


def load_config(k):
    """(PackedH2, extras) for BASELINE config k: data/cfg<k>.npz (full, built by
    tools/make_golden.py) or the committed compact fixtures/cfg<k>.npz; skip if neither."""
    for path in (os.path.join(DATA, f"cfg{k}.npz"), os.path.join(DATA, f"cfg{k}_compact.npz"),
                 os.path.join(ROOT, "fixtures", f"cfg{k}.npz")):
        if os.path.exists(path):
            break
    else:
        pytest.skip(f"cfg{k} operator not present (generate with tools/make_golden.py --configs {k})")
    key = f"cfg{k}"
    if key not in _cache:
        from paper_1703_01175_b200.pack import load_packed
        _cache[key] = load_packed(path, with_extra=True)
    return _cache[key]


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
