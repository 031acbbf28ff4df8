"""Device-side payloads of structure-exact operators (benchmark input preparation).

A structure-exact operator (`pack.save_structure`, tools/make_structures.py) carries the
reference's block structure and ranks but no far-field values; for operators too large to
materialise on the host (BASELINE cfg4: ~35 GB of couplings) the seeded V/T/S values are
generated directly in HBM, chunk by chunk, and copied into the handle's sections through the
ordinary `h2b_upload` (which accepts device sources).  Same value distribution as
`pack._synthetic_far_field`; not the same stream of numbers (no parity claim is made on these
operators — their purpose is bytes, flops and the roofline).
"""

from __future__ import annotations

_CHUNK = 1 << 27  # complex elements per generated chunk (2 GiB)


def fill_far_field_on_device(lib, handle, pk, device, seed):
    import torch

    from . import _abi
    ev, et, es = pk.far_elems_expected()
    gen = torch.Generator(device=f"cuda:{device}")
    gen.manual_seed(int(seed))
    for sec, elems, scale in ((_abi.SEC_V, ev, 0.125), (_abi.SEC_T, et, 0.125), (_abi.SEC_S, es, 0.01)):
        for e0 in range(0, elems, _CHUNK):
            n = min(_CHUNK, elems - e0)
            buf = torch.randn(2 * n, dtype=torch.float64, device=f"cuda:{device}", generator=gen)
            buf.mul_(scale)
            torch.cuda.synchronize(device)
            _abi.check(lib.h2b_upload(handle, sec, buf.data_ptr(), 16 * n, 16 * e0), "h2b_upload")
            del buf
