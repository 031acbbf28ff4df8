"""fixtures/cfg<k>_structure.npz: index tables + geometry of a reference-built BASELINE operator.

Too large to ship whole (cfg3: 7.1 GB; the GPU-box snapshot limit is 512 MiB), the operator
travels as its exact block structure and ranks (from data/cfg<k>.npz, built by the
reference, tools/make_golden.py) — `load_packed` fills seeded far-field payloads and the
near-field is sampled from the geometry on the device.  Throughput, bytes and flops are those
of the reference operator; parity runs against the oracle on the same synthetic payloads.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_fixtures import GEOM  # noqa: E402
from paper_1703_01175_b200.pack import load_packed, save_structure  # noqa: E402

for k in [int(a) for a in sys.argv[1:] or ["3"]]:
    src = os.path.join(ROOT, "data", f"cfg{k}_compact.npz")
    pk = load_packed(src if os.path.exists(src) else os.path.join(ROOT, "data", f"cfg{k}.npz"),
                     near_on_host=False)
    out = os.path.join(ROOT, "fixtures", f"cfg{k}_structure.npz")
    save_structure(pk, out, GEOM[k], seed=k,
                   note=f"block structure and ranks of the reference-built cfg{k}; V/T/S values seeded")
    print(out, os.path.getsize(out) / 1e6, "MB", "B_alg", pk.algorithmic_bytes() / 1e6, "MB")
