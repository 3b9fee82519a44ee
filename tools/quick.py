"""Device-only MLUPS of the default kernels: cavity n^3, three storage modes,
two-buffer and in-place.  usage: python tools/quick.py [n] [steps]"""
import json, os, sys
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
mask = B.flatten_mask(B.cavity_mask(n, n, n))
for prec in (Precision.SINGLE, Precision.DOUBLE, Precision.MIXED1, Precision.MIXED2):
    if os.environ.get("MLB_PRECS") and prec.token not in os.environ["MLB_PRECS"].split(","):
        continue
    for mode in ("ab", "inplace"):
        plan = KernelPlan(n, n, n, Layout.ROW, prec, mask, 1.53, (0.1, 0, 0))
        if os.environ.get("MLB_VARIANT"):
            v = int(os.environ["MLB_VARIANT"])
            plan.set_variant(v if v < 1000 or prec in (Precision.SINGLE, Precision.DOUBLE) else v + 1000)
        if os.environ.get("MLB_PREFETCH"):
            plan.set_prefetch(int(os.environ["MLB_PREFETCH"]))
        a = plan.alloc()
        for q in range(19):
            a.tensor[q].fill_(float(W[q]))
        if mode == "ab":
            b = plan.alloc()
            b.tensor.copy_(a.tensor)
            plan.set_passthrough(True)
            plan.run_steps(a, b, 6)
            _, _, ms = plan.run_steps(a, b, steps, timed=True)
        else:
            b = None
            plan.run_steps_inplace(a, 6)
            ms = plan.run_steps_inplace(a, steps, timed=True)
        ml = n ** 3 * steps / (ms * 1e-3) / 1e6
        gbs = ml * 1e6 * 38 * prec.storage.itemsize / 1e9
        print(json.dumps(dict(n=n, prec=prec.token, mode=mode, kernel=plan.kernel_name if mode == "ab" else "aa",
                              ms_per_step=round(ms / steps, 4), mlups=round(ml), gbs=round(gbs), frac=round(gbs / peak, 4))),
              flush=True)
        plan.close(); del a, b; torch.cuda.empty_cache()
