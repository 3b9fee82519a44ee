"""Where the time of a host-resident run goes: plain upload / download, duplex
PCIe bandwidth, and the overlapped run (mlb_run_steps_host) for several chunk
sizes.  usage: python tools/e2e_host.py [n] [steps]"""
import os, sys, time
sys.path.insert(0, os.environ.get("MLB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.kernels import KernelPlan, pinned_empty
from paper_2409_16781_b200.lattice import W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
prec = Precision.SINGLE
mask = B.flatten_mask(B.cavity_mask(n, n, n))
host = pinned_empty((19, n ** 3), np.float32)
for q in range(19):
    host[q].fill(W[q])
gb = host.nbytes / 1e9
plan = KernelPlan(n, n, n, Layout.ROW, prec, mask, 1.53, (0.1, 0, 0))
a, b = plan.alloc(), plan.alloc()

def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best

t = timed(lambda: plan.upload(host, a)); print(f"upload   {t*1e3:7.1f} ms  {gb/t:5.1f} GB/s")
t = timed(lambda: plan.download(a, host)); print(f"download {t*1e3:7.1f} ms  {gb/t:5.1f} GB/s")
# duplex: one block up while the other comes down, on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
hp = torch.from_numpy(host); hq = torch.empty_like(hp).pin_memory()
da, db = a.tensor[:, 1:-1].reshape(19, -1), b.tensor[:, 1:-1].reshape(19, -1)
def duplex():
    with torch.cuda.stream(s1): da.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2): hq.copy_(db, non_blocking=True)
t = timed(duplex); print(f"duplex   {t*1e3:7.1f} ms  {2*gb/t:5.1f} GB/s both ways")
def up_only():
    with torch.cuda.stream(s1): da.copy_(hp, non_blocking=True)
t = timed(up_only); print(f"torch up {t*1e3:7.1f} ms  {gb/t:5.1f} GB/s")
for k in (0, 1, steps):
    for cz in (0, 2, 8, 32):
        def run():
            plan.run_host(host, host, a, b, k, chunk_planes=cz)
        t = timed(run, 2)
        _, _, ms, ov = plan.run_host(host, host, a, b, k, chunk_planes=cz)
        print(f"run_host K={k:3d} chunk={cz:2d}: wall {t*1e3:7.1f} ms, device {ms:7.1f} ms, overlapped={ov}")
_, _, ms = plan.run_steps(a, b, steps, timed=True)
print(f"{steps} plain steps: {ms:.1f} ms")
