"""Device time of the diagnostics kernels at n^3 (macro: rho,u fields; diag: scalar reductions)."""
import os, sys
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
for prec in (Precision.SINGLE, Precision.DOUBLE, Precision.MIXED1):
    plan = KernelPlan(n, n, n, Layout.ROW, prec, B.flatten_mask(B.cavity_mask(n, n, n)), 1.5, (0.1, 0, 0))
    a = plan.alloc()
    for q in range(19):
        a.tensor[q].fill_(float(W[q]))
    item = prec.storage.itemsize
    for name, fn, nbytes in (("macro", lambda: plan.macro(a), n ** 3 * (19 * item + 32)),
                             ("diag", lambda: plan.diagnostics(a), n ** 3 * (19 * item + 1))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            out = fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{n}^3 {prec.token:7s} {name:5s}: {ms:7.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s algorithmic")
        del out
    plan.close(); del a; torch.cuda.empty_cache()
