"""Scratch perf sweep: block widths x precisions x sizes, device-only MLUPS."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan

def run(n, prec, width, steps=30, omega=1.7):
    nx = ny = nz = n
    mask = B.flatten_mask(B.cavity_mask(nx, ny, nz))
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, mask, omega, (0.1, 0, 0))
    plan.set_variant(width)
    a, b = plan.alloc(), plan.alloc()
    from paper_2409_16781_b200.lattice import W
    for q in range(19):
        a.tensor[q].fill_(float(W[q])); b.tensor[q].fill_(float(W[q]))
    plan.run_steps(a, b, 5)
    _, _, ms = plan.run_steps(a, b, steps, timed=True)
    ml = n**3 * steps / (ms * 1e-3) / 1e6
    bpc = 38 * prec.storage.itemsize
    out = dict(n=n, prec=prec.token, width=width, ms_per_step=ms/steps, mlups=ml, gbs=ml*1e6*bpc/1e9)
    print(json.dumps(out), flush=True)
    plan.close()
    del a, b
    torch.cuda.empty_cache()

if __name__ == "__main__":
    sizes = [int(s) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["256", "512"])]
    for n in sizes:
        for prec in (Precision.SINGLE, Precision.DOUBLE):
            for width in (128, 1008, 1016, 1032):
                run(n, prec, width)
