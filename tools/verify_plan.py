"""Run the planner's schedule self-check (H2B_VERIFY_PLAN) on fixtures / configs."""
import sys, os, glob
os.environ["H2B_VERIFY_PLAN"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_01175_b200 import H2Operator, load_packed, _abi
paths = sys.argv[1:] or sorted(glob.glob("tests/golden/*.npz")) + sorted(glob.glob("data/cfg[12].npz"))
for p in paths:
    pk = load_packed(p)
    op = H2Operator(pk)
    print(p, flush=True)
    _abi.check(_abi.lib().h2b_prepare_handle(op.handle))
    sys.stderr.flush()
