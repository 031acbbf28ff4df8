import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_01175_b200 import gmres_solve, load_packed, H2Operator, _abi
pk, ex = load_packed("data/cfg1.npz", with_extra=True)
b = ex["x"][:, 0]
ho = np.asarray(ex["gmres_hist"])
for mega in (1, 0):
    op = H2Operator(pk)
    _abi.check(_abi.lib().h2b_set_option(op.handle, 2, mega))
    x, rep = gmres_solve(op, b, tol=1e-6, restart=30, max_iter=2000)
    h = np.asarray(rep.residual_history)
    n = min(len(h), len(ho))
    d = np.abs(h[:n] - ho[:n]) / ho[:n]
    first = int(np.argmax(d > 1e-6)) if np.any(d > 1e-6) else -1
    print(f"mega={mega} iters={rep.iterations} first divergence > 1e-6 rel at it {first}; "
          f"max rel diff first 30: {d[:30].max():.2e}, at 60: {d[:60].max():.2e}, at 240: {d[:240].max():.2e}")
    y = op.matvec(ex["x"][:, 1])
    print("   matvec relerr", np.linalg.norm(y - ex["y"][:, 1]) / np.linalg.norm(ex["y"][:, 1]))
    op.close()
