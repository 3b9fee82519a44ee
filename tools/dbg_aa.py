import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from tests.helpers import geometries3d, random_block
geom, tag = sys.argv[1], sys.argv[2]
prec = {"f32": Precision.SINGLE, "f64": Precision.DOUBLE, "f16": Precision.MIXED1}[tag]
grid, wall_u, _ = geometries3d()[geom]
nx, ny, nz = grid.shape
def report(name, got, want):
    g4, w4 = got.reshape(19, nz, ny, nx), want.reshape(19, nz, ny, nx)
    bad = np.argwhere(g4 != w4)
    print(name, "mismatches", len(bad))
    for q, z, y, x in bad[:8]:
        print("   q", q, "x", x, "y", y, "z", z, "flag", grid[x, y, z], repr(g4[q, z, y, x]), repr(w4[q, z, y, x]))
for variant in [int(v) for v in sys.argv[3].split(",")]:
    for steps in (1,):
        rng = np.random.default_rng(20240917)
        f = random_block(rng, grid.size, prec.storage)
        orc = CpuOracle(nx, ny, nz, B.flatten_mask(grid), 1.45, wall_u)
        want = orc.run(f.copy(), f.copy(), steps)
        for mode in ("ab", "aa"):
            plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), 1.45, wall_u)
            plan.set_variant(variant)
            d = plan.alloc(); plan.upload(f, d)
            if mode == "aa":
                plan.run_steps_inplace(d, steps); plan.normalize(d)
            else:
                e = plan.alloc(); plan.upload(f, e)
                d, _, _ = plan.run_steps(d, e, steps)
            got = np.empty_like(f); plan.download(d, got)
            report(f"{geom} {tag} variant {variant} steps {steps} {mode}", got, want)
