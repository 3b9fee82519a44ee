"""Device-only MLUPS of chosen kernel variants, two-buffer, cavity n^3.
usage: python tools/variants.py n steps prec variant [variant ...]   (0 = auto, 4000 = staged)"""
import json, os, sys
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W

n, steps, prec = int(sys.argv[1]), int(sys.argv[2]), Precision.from_token(sys.argv[3])
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
mask = B.flatten_mask(B.cavity_mask(n, n, n))
for v in (int(x) for x in sys.argv[4:]):
    plan = KernelPlan(n, n, n, Layout.ROW, prec, mask, 1.53, (0.1, 0, 0))
    plan.set_variant(v)
    if os.environ.get("MLB_PREFETCH"):
        plan.set_prefetch(int(os.environ["MLB_PREFETCH"]))
    a = plan.alloc()
    for q in range(19):
        a.tensor[q].fill_(float(W[q]))
    b = plan.alloc(); b.tensor.copy_(a.tensor)
    plan.set_passthrough(True)
    plan.run_steps(a, b, 6)
    best = 0.0
    for rep in range(3):
        _, _, ms = plan.run_steps(a, b, steps, timed=True)
        best = max(best, n ** 3 * steps / (ms * 1e-3) / 1e6)
    gbs = best * 1e6 * 38 * prec.storage.itemsize / 1e9
    print(json.dumps(dict(n=n, prec=prec.token, variant=v, kernel=plan.kernel_name, mlups=round(best),
                          frac=round(gbs / peak, 4))), flush=True)
    plan.close(); del a, b; torch.cuda.empty_cache()
