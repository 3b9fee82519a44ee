"""Scratch perf sweep: block widths x precisions x sizes, device-only MLUPS."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan

def run(n, prec, width, steps=30, omega=1.7):
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    mask = B.flatten_mask(B.cavity_mask(nx, ny, nz))
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, mask, omega, (0.1, 0, 0))
    plan.set_variant(width)
    plan.set_passthrough(os.environ.get('PT', '1') == '1')
    a, b = plan.alloc(), plan.alloc()
    from paper_2409_16781_b200.lattice import W
    for q in range(19):
        a.tensor[q].fill_(float(W[q])); b.tensor[q].fill_(float(W[q]))
    plan.run_steps(a, b, 5)
    _, _, ms = plan.run_steps(a, b, steps, timed=True)
    ml = nx * ny * nz * steps / (ms * 1e-3) / 1e6
    bpc = 38 * prec.storage.itemsize
    out = dict(n=n, prec=prec.token, width=width, ms_per_step=ms/steps, mlups=ml, gbs=ml*1e6*bpc/1e9)
    print(json.dumps(out), flush=True)
    plan.close()
    del a, b
    torch.cuda.empty_cache()

def run_inplace(n, prec, steps=30, omega=1.7):
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    mask = B.flatten_mask(B.cavity_mask(nx, ny, nz))
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, mask, omega, (0.1, 0, 0))
    a = plan.alloc()
    from paper_2409_16781_b200.lattice import W
    for q in range(19):
        a.tensor[q].fill_(float(W[q]))
    plan.run_steps_inplace(a, 6)
    ms = plan.run_steps_inplace(a, steps, timed=True)
    ml = nx * ny * nz * steps / (ms * 1e-3) / 1e6
    bpc = 38 * prec.storage.itemsize
    print(json.dumps(dict(n=n, prec=prec.token, mode="inplace", ms_per_step=ms/steps, mlups=ml, gbs=ml*1e6*bpc/1e9)), flush=True)
    plan.close(); del a; torch.cuda.empty_cache()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "inplace":
        for n in (512, 256):
            for prec in (Precision.SINGLE, Precision.DOUBLE, Precision.MIXED1):
                run_inplace(n, prec)
        sys.exit(0)
    sizes = [int(s) if "x" not in s else tuple(int(v) for v in s.split("x"))
             for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["256", "512"])]
    f32v = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [128, 1016, 1116, 2008, 2016, 2032, 2108, 2116, 2132]
    f64v = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [128, 1016, 1116]
    for n in sizes:
        for width in f32v:
            run(n, Precision.SINGLE, width)
        for width in f64v:
            run(n, Precision.DOUBLE, width)
