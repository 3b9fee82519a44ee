import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_16781_b200 import cases, engine
from paper_2409_16781_b200.fields import Precision
n = 512
state = cases.init(cases.CaseSpec("ldc", n, n, n, re=1000.0, u0=0.1), Precision.SINGLE)
for inplace in (False, True, True):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sess = engine.open_session(state, engine.RunConfig(steps=1, inplace=inplace))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        sess.advance(200)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        sess.sync_host()
        t3 = time.perf_counter()
        sess.close(sync=False)
        torch.cuda.synchronize(); t4 = time.perf_counter()
        print(f"inplace={inplace} rep {rep}: open {t1-t0:.3f}  200 steps {t2-t1:.3f}  sync_host {t3-t2:.3f}  close {t4-t3:.3f}  f_post_ is None: {state.f_post_ is None}")
for inplace in (False, True):
    engine.run(state, engine.RunConfig(steps=5, inplace=inplace))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    engine.run(state, engine.RunConfig(steps=200, inplace=inplace))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"engine.run inplace={inplace}: {t1-t0:.3f} s")
    torch.cuda.empty_cache()
    engine.run(state, engine.RunConfig(steps=5, inplace=inplace))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    engine.run(state, engine.RunConfig(steps=200, inplace=inplace))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"after empty_cache: engine.run inplace={inplace}: {t1-t0:.3f} s")
