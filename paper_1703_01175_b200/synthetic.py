"""Seeded payload values of structure-exact operators (benchmark input preparation).

A structure-exact operator (`pack.save_structure`, tools/make_structures.py) carries the
reference's block structure and ranks but no far-field values.  The values come from a
counter-based generator, value(seed, section, global element index) — libh2b's
``h2b_fill_synthetic_*`` on the device, `synth_values` here (bit-identical: integer hashing and
exact conversions only) — so a block has the same values wherever it is materialised: in the
single-GPU handle's V/T/S sections, in any rank's shard payload (`shard.plan_shard(...,
device_payloads=True)`), or on the host for the CPU oracle.  No parity claim is made against
the reference on these operators; they serve bytes, flops and the roofline, and let the
partitioned operator be checked against the single-GPU one element for element.
"""

from __future__ import annotations

import numpy as np

SCALES = (0.125, 0.125, 0.01)  # V, T, S: uniform in [-scale, scale] (re and im)
_CHUNK = 1 << 27               # complex elements per device-generated chunk (2 GiB)
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def synth_values(seed, section, start, n, scale):
    """value(seed, section, start + e) for e < n, as libh2b's k_fill_raw computes it."""
    with np.errstate(over="ignore"):
        idx = np.arange(start, start + n, dtype=np.uint64)
        h = _splitmix64(np.uint64(seed) ^ (np.uint64(section) << np.uint64(56))
                        ^ (idx * np.uint64(0x9E3779B97F4A7C15)))
    u1 = (h >> np.uint64(32)).astype(np.float64) * (1.0 / 4294967296.0)
    u2 = (h & np.uint64(0xFFFFFFFF)).astype(np.float64) * (1.0 / 4294967296.0)
    out = np.empty(n, dtype=np.complex128)
    out.real = (u1 - 0.5) * 2.0 * scale
    out.imag = (u2 - 0.5) * 2.0 * scale
    return out


def host_far_field(pk, seed=None):
    """V, T, S of a structure-exact operator on the host (same values as on the device)."""
    seed = int(pk.meta.get("synthetic", {}).get("seed", 0)) if seed is None else int(seed)
    ev, et, es = pk.far_elems_expected()
    return dict(vbuf=synth_values(seed, 0, 0, ev, SCALES[0]),
                tbuf=synth_values(seed, 1, 0, et, SCALES[1]),
                sbuf=synth_values(seed, 2, 0, es, SCALES[2]))


def fill_far_field_on_device(lib, handle, pk, device, seed):
    """Generate V/T/S in HBM chunk by chunk and copy them into the handle's sections."""
    import ctypes as C

    import torch

    from . import _abi
    ev, et, es = pk.far_elems_expected()
    for sec, elems in ((_abi.SEC_V, ev), (_abi.SEC_T, et), (_abi.SEC_S, es)):
        buf = torch.empty(min(_CHUNK, max(elems, 1)), dtype=torch.complex128, device=f"cuda:{device}")
        for e0 in range(0, elems, _CHUNK):
            n = min(_CHUNK, elems - e0)
            _abi.check(lib.h2b_fill_synthetic_raw(C.c_void_p(buf.data_ptr()), n, e0, sec, int(seed),
                                                  SCALES[sec]), "h2b_fill_synthetic_raw")
            _abi.check(lib.h2b_upload(handle, sec, buf.data_ptr(), 16 * n, 16 * e0), "h2b_upload")
        del buf
