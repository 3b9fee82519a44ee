import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2409_16781_b200 import boundaries as B, cases
from paper_2409_16781_b200 import lattice as L
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
nx, ny, nz = 1024, 512, 512
spec = cases.CaseSpec("vks", nx, ny, nz, re=200.0, u0=0.08)
flags = B.flatten_mask(spec.mask())
plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE, flags, spec.relaxation().omega, inlet_u=0.08)
plan.set_passthrough(os.environ.get("PT", "1") == "1")
eq = L.equilibrium(1.0, 0.08, 0.0, 0.0).astype(np.float32)
a = plan.alloc()
for q in range(19):
    a.tensor[q].fill_(float(eq[q]))
b = plan.alloc(); b.tensor.copy_(a.tensor)
plan.run_steps(a, b, 4)
_, _, ms = plan.run_steps(a, b, 20, timed=True)
print(f"channel: {nx*ny*nz*20/ms/1e3:.0f} MLUPS, {ms/20:.3f} ms/step")
# the same channel in place (one block): bit-compare with the two-buffer result
import torch
newest = a  # 24 steps (even) end in a
c = plan.alloc()
for q in range(19):
    c.tensor[q].fill_(float(eq[q]))
plan.run_steps_inplace(c, 4)
ms = plan.run_steps_inplace(c, 20, timed=True)
plan.normalize(c)
same = bool(torch.equal(c.tensor[:, 1:-1], newest.tensor[:, 1:-1]))
print(f"channel in place: {nx*ny*nz*20/ms/1e3:.0f} MLUPS, {ms/20:.3f} ms/step, equals two-buffer result bitwise: {same}")
