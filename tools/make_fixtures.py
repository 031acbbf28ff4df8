"""Write the committed, compact copies of the BASELINE operators: fixtures/cfg<k>.npz.

data/cfg<k>.npz (tools/make_golden.py --configs k, needs the reference) holds the
full packed operator.  The fixture drops the near-field payload, which is a
plain sample of the system matrix, and records the geometry instead;
`pack.load_packed` re-assembles it (nearfield.py).  Before writing, the
re-assembled payload is checked against the reference-built one.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1703_01175_b200.nearfield import assemble_near, geometry_arrays  # noqa: E402
from paper_1703_01175_b200.pack import load_packed, save_packed  # noqa: E402

GEOM = {
    1: dict(kind="lattice", dims=[16, 16, 16], h=1.0 / 16, eps_r=4.0, k0=2 * np.pi),
    2: dict(kind="lattice", dims=[65536, 1, 1], h=1.0 / 32, eps_r=4.0, k0=2 * np.pi),
    3: dict(kind="lattice", dims=[512, 512, 1], h=1.0 / 16, eps_r=4.0, k0=2 * np.pi),
}

def main():
    for k in [int(a) for a in (sys.argv[1:] or ["1", "2"])]:
        pk, ex = load_packed(os.path.join(ROOT, "data", f"cfg{k}.npz"), with_extra=True)
        d = assemble_near(pk, *geometry_arrays(GEOM[k]))
        err = np.max(np.abs(d - pk.dbuf)) / np.max(np.abs(pk.dbuf))
        print(f"cfg{k}: re-assembled near-field max rel deviation {err:.2e}")
        assert err < 1e-13
        keep = dict(ex)
        # cfg3 (1.7 GB without its near-field) is too large to commit or ship:
        # data/cfg3_compact.npz stays local; fixtures/cfg3_structure.npz travels
        out = (os.path.join(ROOT, "fixtures", f"cfg{k}.npz") if k < 3
               else os.path.join(ROOT, "data", f"cfg{k}_compact.npz"))
        save_packed(pk, out, extra=keep, geometry=GEOM[k])
        print(f"  -> {out} {os.path.getsize(out) / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
