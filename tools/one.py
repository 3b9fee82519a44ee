"""Run a few steps of one configuration (for ncu captures)."""
import sys, os
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W
nx, ny, nz = (int(v) for v in sys.argv[1].split("x"))
prec = Precision.from_token(sys.argv[2])
variant = int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
case = sys.argv[5] if len(sys.argv) > 5 else "cavity"
grid = B.cavity_mask(nx, ny, nz) if case == "cavity" else B.open_mask(nx, ny, nz)
plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), 1.7, (0.1, 0, 0))
plan.set_variant(variant)
plan.set_passthrough(os.environ.get('PT', '1') == '1')
a, b = plan.alloc(), plan.alloc()
for q in range(19):
    a.tensor[q].fill_(float(W[q])); b.tensor[q].fill_(float(W[q]))
_, _, ms = plan.run_steps(a, b, steps, timed=True)
print(f"{nx}x{ny}x{nz} {prec.token} v{variant} {case}: {nx*ny*nz*steps/ms/1e3:.0f} MLUPS")
