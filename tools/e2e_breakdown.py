import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import cases, engine
from paper_2409_16781_b200.fields import Precision
n = 512
t0 = time.perf_counter()
state = cases.init(cases.CaseSpec("ldc", n, n, n, re=1000.0, u0=0.1), Precision.SINGLE)
print(f"host init (pinned alloc + fill): {time.perf_counter()-t0:.3f} s")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    plan = engine.build_plan(state, engine.RunConfig(steps=1))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    sess = engine.Session(state, plan)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    sess.advance(200)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    sess.sync_host()
    t4 = time.perf_counter()
    sess.close(sync=False)
    print(f"rep {rep}: plan {t1-t0:.3f}  alloc+upload {t2-t1:.3f} ({10.24/(t2-t1):.1f} GB/s incl. D2D copy)  200 steps {t3-t2:.3f}  download {t4-t3:.3f} ({10.2/(t4-t3):.1f} GB/s)")
