"""B200-native (sm_100a) H² matvec + Krylov hot path behind the `h2vie` operator API.

Drop-in surface (mirrors /root/reference/pkg/src/h2vie/__init__.py:8-17 for
the hot path only):

    matvec(h2, x)                       arith.py:108-117
    matmat_apply(h2, X, col_block=256)  arith.py:120-130
    bicgstab_solve(apply, rhs, ...)     arith.py:605-689
    gmres_solve(apply, rhs, ...)        new (the reference has no GMRES)
    block_gmres_solve(apply, rhs, ...)  new: q right-hand sides (BASELINE config 5)
    SolveReport                         arith.py:39-44

``h2`` is a reference ``H2Matrix`` (packed on first use) or a `PackedH2`
loaded from disk (`load_packed`).  Everything numeric runs in libh2b.so.
"""

from .pack import PackedH2, load_packed, pack_h2, save_packed, validate
from .h2op import H2Operator, as_operator, matmat_apply, matvec
from .krylov import SolveReport, bicgstab_solve, gmres_solve
from .block_krylov import block_gmres_solve

__all__ = [
    "PackedH2", "load_packed", "pack_h2", "save_packed", "validate",
    "H2Operator", "as_operator", "matmat_apply", "matvec",
    "SolveReport", "bicgstab_solve", "gmres_solve", "block_gmres_solve",
]

__version__ = "0.1.0"
