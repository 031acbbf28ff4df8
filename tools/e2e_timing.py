import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1703_01175_b200 import as_operator, matvec
from paper_1703_01175_b200.pack import load_packed
pk, ex = load_packed("fixtures/cfg2.npz", with_extra=True)
x = ex["x"][:, 0].copy()
for _ in range(30): matvec(pk, x)
