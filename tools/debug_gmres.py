import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_01175_b200 import gmres_solve, load_packed
pk, ex = load_packed("tests/golden/rod164.npz", with_extra=True)
try:
    x, rep = gmres_solve(pk, ex["x"][:, 0], tol=1e-8, restart=30, max_iter=2000)
    print(rep.iterations, rep.converged)
except Exception as e:
    print("ERR", e)
