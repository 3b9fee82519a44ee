import os, sys, signal
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
def worker(rank, world, port):
    signal.alarm(200)
    import torch, torch.distributed as dist
    from paper_2409_16781_b200 import cases, engine
    from paper_2409_16781_b200.fields import Precision
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = cases.CaseSpec("ldc", 128, 12, 9, re=100.0, u0=0.1)
    probe = (60, 10, 5)
    alone = cases.init(spec, Precision.SINGLE)
    ra = engine.run(alone, engine.RunConfig(steps=9, distributed=False), probe=probe)
    for inplace in (False, True):
        st = cases.init(spec, Precision.SINGLE)
        rs = engine.run(st, engine.RunConfig(steps=9, inplace=inplace), probe=probe)
        if rank == 0:
            bad = np.argwhere(rs.probe_samples != ra.probe_samples)
            print("inplace", inplace, "state equal", np.array_equal(st.f_pre.data, alone.f_pre.data), "probe mismatches", bad.tolist()[:12])
            print(rs.probe_samples[:4], ra.probe_samples[:4])
    dist.destroy_process_group()
if __name__ == "__main__":
    import torch.multiprocessing as mp
    mp.spawn(worker, args=(2, 29533), nprocs=2, join=True)
