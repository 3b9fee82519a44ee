"""The fused peer-store halo exchange across PROCESSES: two or three ranks,
each with its own CUDA context, map each other's population blocks and step
counters through CUDA IPC and run the real DistSlab + PeerRing driver.  On a
box with enough GPUs every rank takes its own device (rank % device_count,
NCCL control plane) and the stores cross NVLink; on a one-GPU box all ranks
share device 0 - the memory mapping, the in-kernel stores into the
neighbour's halo planes and the stream-ordered signal protocol are exactly
what runs with one rank per GPU; only the wire differs - with a gloo control
plane (helpers.init_ranks).  The gathered result must be BITWISE the
single-domain run."""

import os
import signal
import socket

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision

from .helpers import geometries3d, init_ranks, random_block

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, geom, tag, steps, omega, wait_mode, overlap, passthrough, out_dir,
            c_loop=True):
    signal.alarm(240)  # a protocol bug must not hang the box
    import torch.distributed as dist
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    _, fdev = init_ranks(rank, world, port)
    try:
        grid, wall_u, inlet_u = geometries3d()[geom]
        prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE, "f16": Precision.MIXED1}[tag]
        nx, ny, nz = grid.shape
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        f = random_block(np.random.default_rng(20240917), grid.size, prec.storage)
        z0, z1 = slab.partition(nz, world)[rank]
        n = z1 - z0
        lo, hi = slab.exchange_flag_halos(flags[z0:z1], rank, world, device=fdev)
        plan = KernelPlan(nx, ny, n, Layout.ROW, prec, flags[z0:z1], omega, wall_u,
                          inlet_u=inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
        part = np.ascontiguousarray(f.reshape(19, nz, ny, nx)[:, z0:z1]).reshape(19, -1)
        blocks = [plan.alloc(), plan.alloc()]
        for blk in blocks:
            blk.tensor.fill_(float("nan"))
            plan.upload(part, blk)
        if passthrough:
            try:
                plan.set_passthrough(True)
            except ValueError:
                pass
        ring = slab.PeerRing(plan, blocks, rank, world, wait_mode=wait_mode)
        runner = slab.DistSlab(slab.CudaStepper(plan), n, rank, world, overlap=overlap, ring=ring,
                               c_loop=c_loop)
        runner.exchange(blocks[0])
        newest, _ = runner.run(blocks[0], blocks[1], steps)
        runner.finish()
        out = np.empty_like(part)
        plan.download(newest, out)
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), out.reshape(19, n, ny, nx))
        ring.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wait_mode,c_loop", [(0, True), (2, True), (0, False)])
@pytest.mark.parametrize("geom,tag,world,overlap,passthrough", [
    ("cavity_oblique_lid", "f64", 2, False, False),
    ("cavity16", "f32", 2, True, True),
    ("channel40", "f32", 2, True, True),
    ("channel", "f64", 3, True, False),
    ("open_unfusable", "f32", 2, False, True),
    ("periodic8", "f16", 2, False, True),
    ("cavity16", "f32", 3, False, True),
])
def test_peer_ring_across_processes(geom, tag, world, overlap, passthrough, wait_mode, c_loop,
                                    tmp_path):
    """c_loop: the whole loop in one library call (mlb_slab_run_steps, the
    default) or the same schedule driven step by step from Python."""
    import torch.multiprocessing as mp
    steps, omega = 7, 1.3
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    dtype = {"f64": np.float64, "f32": np.float32, "f16": np.float16}[tag]
    f = random_block(np.random.default_rng(20240917), grid.size, dtype)
    want = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u).run(
        f.copy(), f.copy(), steps)
    mp.spawn(_worker, args=(world, _free_port(), geom, tag, steps, omega, wait_mode, overlap,
                            passthrough, str(tmp_path), c_loop), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=1)
    np.testing.assert_array_equal(got.reshape(19, -1), want)


def _nccl_worker(rank, port, geom, steps, omega, out_dir):
    signal.alarm(240)
    import torch
    import torch.distributed as dist
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        f = random_block(np.random.default_rng(20240917), grid.size, np.float32)
        lo, hi = slab.exchange_flag_halos(flags, 0, 1)
        plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE, flags, omega, wall_u,
                          inlet_u=inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
        blocks = [plan.alloc(), plan.alloc()]
        for blk in blocks:
            blk.tensor.fill_(float("nan"))
            plan.upload(f, blk)
        runner = slab.DistSlab(slab.CudaStepper(plan), nz, 0, 1, force_dist=True)
        for r in runner.exchange(blocks[0]):
            r.wait()
        newest, _ = runner.run(blocks[0], blocks[1], steps)
        out = np.empty_like(f)
        plan.download(newest, out)
        np.save(os.path.join(out_dir, "nccl.npy"), out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("geom", ["cavity16", "channel40"])
def test_send_recv_transport_over_nccl(geom, tmp_path):
    """The send/recv fallback on the real NCCL backend: one rank whose ring
    closes on itself THROUGH torch.distributed (batch_isend_irecv of the ten
    crossing planes, boundary-first overlap on the high-priority stream)."""
    import torch.multiprocessing as mp
    steps, omega = 6, 1.3
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    f = random_block(np.random.default_rng(20240917), grid.size, np.float32)
    want = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u).run(
        f.copy(), f.copy(), steps)
    mp.spawn(_nccl_worker, args=(_free_port(), geom, steps, omega, str(tmp_path)),
             nprocs=1, join=True)
    np.testing.assert_array_equal(np.load(tmp_path / "nccl.npy"), want)


def _engine_worker(rank, world, port, case, tag, out_dir, inplace=False):
    signal.alarm(240)
    import torch.distributed as dist
    from paper_2409_16781_b200 import cases, engine
    init_ranks(rank, world, port)
    try:
        prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE}[tag]
        spec = (cases.CaseSpec("ldc", 24, 20, 17, re=100.0, u0=0.1) if case == "ldc"
                else cases.CaseSpec("ldc", 128, 12, 9, re=100.0, u0=0.1) if case == "ldc128"
                else cases.CaseSpec("vks", 128, 32, 7, re=100.0, u0=0.08) if case == "vks128"
                else cases.CaseSpec("vks", 48, 32, 11, re=100.0, u0=0.08))
        probe = {"ldc": (12, 10, 9), "ldc128": (60, 10, 5), "vks128": (90, 16, 2)}.get(
            case, (30, 16, 2))
        # the same driver code twice: once alone on this GPU, once as one of `world` slabs
        alone = cases.init(spec, prec)
        seen_alone = []
        ra = engine.run(alone, engine.RunConfig(steps=23, precision=prec, output_every=10,
                                                distributed=False),
                        on_output=lambda st: seen_alone.append((st.t, st.f_pre.data.copy())),
                        probe=probe)
        state = cases.init(spec, prec)
        seen = []
        rs = engine.run(state, engine.RunConfig(steps=23, precision=prec, output_every=10,
                                                inplace=inplace),
                        on_output=lambda st: seen.append((st.t, st.f_pre.data.copy())),
                        probe=probe)
        assert rs.transport == "peer", rs.transport
        assert state.t == alone.t == 23
        np.testing.assert_array_equal(state.f_pre.data, alone.f_pre.data)   # gathered: whole state
        assert [t for t, _ in seen] == [t for t, _ in seen_alone] == [10, 20]
        for (_, x), (_, y) in zip(seen, seen_alone):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(rs.probe_samples, ra.probe_samples)
        open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,tag,world,inplace", [
    ("ldc", "f64", 2, False), ("ldc", "f32", 3, False), ("vks", "f32", 2, False),
    ("ldc128", "f32", 2, True), ("vks128", "f32", 3, True)])
def test_engine_run_is_the_same_call_under_torch_distributed(case, tag, world, inplace, tmp_path):
    """The reference's driver call, unchanged, with one rank per slab: with a
    process group initialised, engine.run splits the domain into z-slabs, runs
    the fused peer-store exchange, fires the hooks at the same cadence with the
    whole host state gathered, and ends bit-identical to the single-GPU run."""
    import torch.multiprocessing as mp
    mp.spawn(_engine_worker, args=(world, _free_port(), case, tag, str(tmp_path), inplace),
             nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


def _inplace_worker(rank, world, port, geom, tag, variant, steps, overlap, wait_mode, out_dir,
                    c_loop=True):
    signal.alarm(240)
    import torch.distributed as dist
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    _, fdev = init_ranks(rank, world, port)
    try:
        grid, wall_u, inlet_u = geometries3d()[geom]
        prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE, "f16": Precision.MIXED1}[tag]
        nx, ny, nz = grid.shape
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        f = random_block(np.random.default_rng(20240917), grid.size, prec.storage)
        z0, z1 = slab.partition(nz, world)[rank]
        n = z1 - z0
        lo, hi = slab.exchange_flag_halos(flags[z0:z1], rank, world, device=fdev)
        plan = KernelPlan(nx, ny, n, Layout.ROW, prec, flags[z0:z1], 1.3, wall_u,
                          inlet_u=inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
        plan.set_variant(variant)
        part = np.ascontiguousarray(f.reshape(19, nz, ny, nx)[:, z0:z1]).reshape(19, -1)
        blk = plan.alloc()
        blk.tensor.fill_(float("nan"))
        plan.upload(part, blk)
        ring = slab.PeerRing(plan, [blk], rank, world, wait_mode=wait_mode)
        runner = slab.DistSlab(slab.CudaStepper(plan), n, rank, world, overlap=overlap, ring=ring,
                               c_loop=c_loop)
        runner.exchange(blk)
        runner.run_inplace(blk, steps)
        runner.normalize(blk)
        out = np.empty_like(part)
        plan.download(blk, out)
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), out.reshape(19, n, ny, nx))
        ring.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("geom,tag,variant,world,steps,overlap,wait_mode,c_loop", [
    ("cavity16", "f32", 1008, 2, 7, False, 0, True),
    ("cavity16", "f32", 1016, 2, 6, True, 2, True),
    ("porous", "f64", 1008, 3, 5, False, 0, True),
    ("channel40", "f32", 1008, 2, 7, False, 0, False),
    ("periodic8", "f16", 2008, 2, 4, False, 0, True),
    ("porous", "f32", 1008, 2, 9, True, 0, False),
])
def test_inplace_slabs_across_processes(geom, tag, variant, world, steps, overlap, wait_mode,
                                        c_loop, tmp_path):
    """One block per rank: the in-place update over z-slabs, ranks in separate
    processes writing into each other's boundary planes (pull half) and halo
    planes (local half) through CUDA IPC mappings."""
    import torch.multiprocessing as mp
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    dtype = {"f64": np.float64, "f32": np.float32, "f16": np.float16}[tag]
    f = random_block(np.random.default_rng(20240917), grid.size, dtype)
    want = CpuOracle(nx, ny, nz, B.flatten_mask(grid), 1.3, wall_u, inlet_u).run(
        f.copy(), f.copy(), steps)
    mp.spawn(_inplace_worker, args=(world, _free_port(), geom, tag, variant, steps, overlap,
                                    wait_mode, str(tmp_path), c_loop), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=1)
    np.testing.assert_array_equal(got.reshape(19, -1), want)


def _chained_worker(rank, world, port, tag, out_dir):
    signal.alarm(240)
    import torch.distributed as dist
    from paper_2409_16781_b200 import engine
    from paper_2409_16781_b200.fields import PopulationField
    from paper_2409_16781_b200.lattice import RelaxationParams
    init_ranks(rank, world, port)
    try:
        prec = {"f32": Precision.SINGLE, "m2": Precision.MIXED2}[tag]
        grid = B.open_mask(16, 6, 9)
        grid[5, 1:5, :] = B.INLET
        grid[13:16, 2:4, 1:8] = B.OUTLET        # three outlet cells in a row: chained
        grid[9, 3, 2] = B.SOLID
        grid[:, 0, :] = B.SOLID
        nx, ny, nz = grid.shape
        mask = B.flatten_mask(grid)
        f = random_block(np.random.default_rng(11), grid.size, prec.storage)
        state = engine.SimState(
            f_pre=PopulationField(f.copy(), nx, ny, nz, Layout.ROW), f_post_=None, mask=mask,
            nx=nx, ny=ny, nz=nz, layout=Layout.ROW, precision=prec,
            params=RelaxationParams.from_omega(1.1), wall_u=(0.0, 0.0, 0.0), inlet_u=0.04)
        # one run cut into three distributed runs, then two steps alone on this GPU
        for k in (3, 4, 2):
            rs = engine.run(state, engine.RunConfig(steps=k, precision=prec))
            assert rs.transport == "peer", rs.transport
        assert state.f_post_ is not None            # the second buffer came back with the first
        engine.run(state, engine.RunConfig(steps=2, precision=prec, distributed=False))
        want = CpuOracle(nx, ny, nz, mask, 1.1, (0.0, 0.0, 0.0), 0.04,
                         compute=np.float64 if prec is Precision.MIXED2 else None).run(
            f.copy(), f.copy(), 11)
        np.testing.assert_array_equal(state.f_pre.data, want)
        open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tag,world", [("f32", 2), ("m2", 3)])
def test_chained_outlets_carry_the_second_block_between_distributed_runs(tag, world, tmp_path):
    """Chained outlet cells read stale values of the SECOND buffer
    (engine.py:179-180 of the reference), so a run cut into several
    engine.run calls must carry it - under a process group too: every rank
    brings its slab of both blocks back to the (gathered) host arrays and the
    next run uploads both.  Ends bitwise on the oracle's unbroken run."""
    import torch.multiprocessing as mp
    mp.spawn(_chained_worker, args=(world, _free_port(), tag, str(tmp_path)), nprocs=world,
             join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


def test_peer_ring_does_not_depend_on_the_torch_allocator(tmp_path, monkeypatch):
    """The population blocks are cudaMalloc memory from the library
    (KernelPlan.alloc -> mlb_block_alloc), so they can be exported over CUDA IPC
    even when torch's caching allocator runs with expandable segments (whose
    blocks cannot): engine.run over 2 ranks still takes the peer-memory ring
    (the worker asserts transport == "peer")."""
    import torch.multiprocessing as mp
    monkeypatch.setenv("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    mp.spawn(_engine_worker, args=(2, _free_port(), "ldc", "f32", str(tmp_path), False),
             nprocs=2, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(2))


def _random_worker(rank, world, port, seeds, out_dir):
    """Many random cases through ONE set of processes: per case a fresh plan, ring
    (IPC handles exchanged and mapped anew) and runner; rank 0 gathers and compares."""
    signal.alarm(420)
    import torch.distributed as dist
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    from .test_gpu_fuzz import PREC, draw_case
    _, fdev = init_ranks(rank, world, port)
    bad = []
    try:
        for seed in seeds:
            tag, grid, omega, wall_u, inlet_u, variant, steps = draw_case(seed)
            prec = PREC[tag]
            nx, ny, nz = grid.shape
            if nz < world:
                continue
            flags = B.flatten_mask(grid).reshape(nz, ny, nx)
            f = random_block(np.random.default_rng(1000 + seed), grid.size, prec.storage)
            z0, z1 = slab.partition(nz, world)[rank]
            n = z1 - z0
            lo, hi = slab.exchange_flag_halos(flags[z0:z1], rank, world, device=fdev)
            plan = KernelPlan(nx, ny, n, Layout.ROW, prec, flags[z0:z1], omega, wall_u,
                              inlet_u=inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
            plan.set_variant(variant if variant != 4000 or seed % 2 else 0)
            part = np.ascontiguousarray(f.reshape(19, nz, ny, nx)[:, z0:z1]).reshape(19, -1)
            inplace = seed % 3 == 0 and 1000 <= variant < 4000
            blocks = [plan.alloc()] if inplace else [plan.alloc(), plan.alloc()]
            for blk in blocks:
                blk.tensor.fill_(float("nan"))
                plan.upload(part, blk)
            if not inplace:
                try:
                    plan.set_passthrough(True)
                except ValueError:
                    pass
            served = True
            if inplace:
                try:    # (raises on EVERY rank if some rank's slab cannot be served in place)
                    runner = slab.open_inplace_runner(plan, blocks[0], rank, world,
                                                      overlap=bool(seed % 2))
                    runner.c_loop = bool(seed % 7)
                    runner.run_inplace(blocks[0], steps)
                    runner.normalize(blocks[0])
                    newest, ring = blocks[0], runner.ring
                except ValueError:
                    served, ring = False, None
            else:
                ring = slab.PeerRing(plan, blocks, rank, world, wait_mode=2 if seed % 5 == 0 else 0)
                runner = slab.DistSlab(slab.CudaStepper(plan), n, rank, world,
                                       overlap=bool(seed % 2), ring=ring, c_loop=bool(seed % 7))
                runner.exchange(blocks[0])
                newest, _ = runner.run(blocks[0], blocks[1], steps)
                runner.finish()
            out = np.empty_like(part)
            if served:
                plan.download(newest, out)
            if ring is not None:
                ring.close()
            plan.close()
            parts = [None] * world
            dist.all_gather_object(parts, out.reshape(19, n, ny, nx))
            if rank == 0 and served:
                got = np.concatenate(parts, axis=1).reshape(19, -1)
                want = CpuOracle(nx, ny, nz, flags, omega, wall_u, inlet_u,
                                 compute=np.float64 if prec is Precision.MIXED2 else None).run(
                    f.copy(), f.copy(), steps)
                if not np.array_equal(got, want):
                    bad.append(seed)
        if rank == 0:
            open(os.path.join(out_dir, "bad.txt"), "w").write(" ".join(map(str, bad)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_ring_random_cases_across_processes(world, tmp_path):
    """The fuzz suite's random cases (shapes, flags incl. chained outlets, dtypes,
    variants) through the peer ring ACROSS processes: two blocks and in place,
    overlap on / off, one-call loop and Python schedule, both wait mechanisms.
    MLB_RING_CASES (default 16) cases per world size through one set of processes."""
    import torch.multiprocessing as mp
    n = int(os.environ.get("MLB_RING_CASES", "16"))
    mp.spawn(_random_worker, args=(world, _free_port(), list(range(500, 500 + n)), str(tmp_path)),
             nprocs=world, join=True)
    assert open(tmp_path / "bad.txt").read().strip() == ""


def _random_engine_worker(rank, world, port, seeds, out_dir):
    """Random cases through the DRIVER call under a process group: per case two
    or three engine.run calls (two blocks / in place, with output hooks), the
    oracle carrying both of its buffers along; every rank holds the gathered
    state and compares."""
    signal.alarm(420)
    import torch.distributed as dist
    from paper_2409_16781_b200 import engine
    from paper_2409_16781_b200.fields import PopulationField
    from paper_2409_16781_b200.lattice import RelaxationParams
    from .test_gpu_fuzz import PREC, draw_case
    init_ranks(rank, world, port)
    bad, ran, refused = [], 0, 0
    try:
        for seed in seeds:
            tag, grid, omega, wall_u, inlet_u, _, _ = draw_case(seed)
            if omega == 0.0:
                omega = 0.7
            prec = PREC[tag]
            nx, ny, nz = grid.shape
            if nz < world:
                continue
            mask = B.flatten_mask(grid)
            r = np.random.default_rng(3000 + seed)
            f = random_block(r, grid.size, prec.storage)
            orc = CpuOracle(nx, ny, nz, mask, omega, wall_u, inlet_u,
                            compute=np.float64 if prec is Precision.MIXED2 else None)
            pre, post = f.copy(), f.copy()
            state = engine.SimState(
                f_pre=PopulationField(f.copy(), nx, ny, nz, Layout.ROW), f_post_=None, mask=mask,
                nx=nx, ny=ny, nz=nz, layout=Layout.ROW, precision=prec,
                params=RelaxationParams.from_omega(omega), wall_u=wall_u, inlet_u=inlet_u)
            for _ in range(int(r.integers(2, 4))):
                k = int(r.integers(1, 8))
                inplace = bool(r.integers(0, 2))
                every = int(r.integers(0, 3))
                seen = []
                try:
                    engine.run(state, engine.RunConfig(steps=k, precision=prec, inplace=inplace,
                                                       output_every=every),
                               on_output=(lambda st: seen.append(st.t)) if every else None)
                except ValueError:      # refused on EVERY rank, before any step
                    refused += 1
                    continue
                ran += 1
                newest = orc.run(pre, post, k)
                if newest is not pre:
                    pre, post = post, pre
                if not np.array_equal(state.f_pre.data, pre):
                    bad.append(seed)
        open(os.path.join(out_dir, f"bad{rank}.txt"), "w").write(
            f"{ran} {refused} " + " ".join(map(str, bad)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_engine_run_random_cases_across_processes(world, tmp_path):
    """The fuzz suite's random cases through engine.run under torch.distributed:
    runs cut into pieces, two blocks and in place, hooks, chained outlet cells
    (the second block travels).  MLB_RING_CASES (default 16) cases per world size."""
    import torch.multiprocessing as mp
    n = int(os.environ.get("MLB_RING_CASES", "16"))
    mp.spawn(_random_engine_worker, args=(world, _free_port(), list(range(800, 800 + n)),
                                          str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ran, refused, *bad = open(tmp_path / f"bad{r}.txt").read().split()
        assert not bad, bad
        assert int(ran) > 0
