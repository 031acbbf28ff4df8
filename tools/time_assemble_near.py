import sys, time, ctypes as C, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1703_01175_b200 import _abi, H2Operator
from paper_1703_01175_b200.pack import load_packed
from paper_1703_01175_b200.nearfield import geometry_arrays, self_term
pk = load_packed("/root/repo/fixtures/cfg5_structure.npz", near_on_host=False, far_on_host=False)
op = H2Operator(pk)  # includes one assembly
L = _abi.lib()
centers, chi, k0, vol = geometry_arrays(pk.meta["geometry"])
diag = k0 ** 2 * self_term(vol, k0)
torch.cuda.synchronize()
for _ in range(3):
    t = time.perf_counter()
    _abi.check(L.h2b_assemble_near(op.handle, centers.ctypes.data, chi.ctypes.data, float(k0), float(vol), float(diag.real), float(diag.imag)))
    dt = time.perf_counter() - t
    print(f"assemble near-field {16*pk.d_elems_expected()/1e9:.1f} GB ({pk.d_elems_expected()/1e6:.0f} M elements): {dt*1e3:.1f} ms incl. host->device of centers/chi")
