"""MLUPS of small, launch-bound domains with and without the CUDA-graph replay
of mlb_run_steps (mlb_plan_set_graph), two-buffer and in place, and a bit
comparison of the two.  usage: python tools/small_domains.py [steps]"""
import json, os, sys
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan
from paper_2409_16781_b200.lattice import W

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for n in (32, 64, 128, 256):
    mask = B.flatten_mask(B.cavity_mask(n, n, n))
    for prec in (Precision.DOUBLE, Precision.SINGLE):
        for mode in ("ab", "inplace"):
            res, bits = {}, {}
            for graph in (0, 1):
                plan = KernelPlan(n, n, n, Layout.ROW, prec, mask, 1.6, (0.1, 0, 0))
                plan.set_graph(graph)
                a = plan.alloc()
                for q in range(19):
                    a.tensor[q].fill_(float(W[q]))
                if mode == "ab":
                    b = plan.alloc(); b.tensor.copy_(a.tensor)
                    plan.set_passthrough(True)
                    plan.run_steps(a, b, 64)
                    _, _, ms = plan.run_steps(a, b, steps, timed=True)
                else:
                    b = None
                    plan.run_steps_inplace(a, 64)
                    ms = plan.run_steps_inplace(a, steps, timed=True)
                    plan.normalize(a)
                res[graph] = n ** 3 * steps / (ms * 1e-3) / 1e6
                bits[graph] = a.tensor[:, 1:-1].clone()
                us = ms * 1e3 / steps
                if graph:
                    same = bool(torch.equal(bits[0], bits[1]))
                    print(json.dumps(dict(n=n, prec=prec.token, mode=mode, steps=steps,
                                          mlups_plain=round(res[0]), mlups_graph=round(res[1]),
                                          speedup=round(res[1] / res[0], 2), us_per_step_graph=round(us, 2),
                                          same_bits=same)), flush=True)
                plan.close(); del a, b
