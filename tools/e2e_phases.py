"""Where does engine.run's fixed cost go?  Phases of 12 back-to-back sessions."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import cases, engine
from paper_2409_16781_b200.fields import Precision
n = 512
state = cases.init(cases.CaseSpec("ldc", n, n, n, re=1000.0, u0=0.1), Precision.SINGLE)
def sync(): torch.cuda.synchronize()
def T(): return time.perf_counter()
for rep in range(12):
    sync(); t = [T()]
    plan = engine.build_plan(state, engine.RunConfig(steps=1), defer_flags=True); sync(); t.append(T())
    a = plan.alloc(); b = plan.alloc(); sync(); t.append(T())
    plan.upload(state.f_pre.data, a); t.append(T())           # enqueue only
    plan.ensure_flags(); t.append(T())
    sync(); t.append(T())
    b.tensor.copy_(a.tensor); plan.set_passthrough(True); sync(); t.append(T())
    plan.run_steps(a, b, 50); sync(); t.append(T())
    plan.download(a, state.f_pre.data); t.append(T())
    plan.close(); sync(); t.append(T())
    del a, b; sync(); t.append(T())
    names = ["plan", "alloc", "upload-enq", "flags", "upload-wait", "d2d", "50steps", "download", "close", "del"]
    d = [t[i + 1] - t[i] for i in range(len(names))]
    print(f"rep {rep:2d} total {t[-1]-t[0]:.3f}: " + "  ".join(f"{k} {v*1e3:.0f}" for k, v in zip(names, d)), flush=True)
