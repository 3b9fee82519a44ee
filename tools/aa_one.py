"""A few in-place steps of the 512^3 cavity (for ncu captures).  usage: aa_one.py [precision] [layout]"""
import sys, os
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W
n = 512
prec = Precision.from_token(sys.argv[1]) if len(sys.argv) > 1 else Precision.SINGLE
plan = KernelPlan(n, n, n, Layout.ROW, prec, B.flatten_mask(B.cavity_mask(n, n, n)), 1.7, (0.1, 0, 0))
if len(sys.argv) > 2:
    plan.set_inplace_layout(int(sys.argv[2]))
a = plan.alloc()
for q in range(19):
    a.tensor[q].fill_(float(W[q]))
plan.run_steps_inplace(a, 8)
