"""The N > 1 path on CPU: two processes, `gloo`, the real DistSlab driver
(partition, flag-halo exchange at setup, per-step 5-population exchange,
ring order) with the CPU oracle as the stepper.  The gathered result must be
BITWISE the single-domain run - the reference's partition-independence
property (test_kernels.py:107-126) carried to z-slabs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.cpu import CpuOracle, SlabOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import slab

from .helpers import geometries3d, random_block


class OracleStepper:
    """CPU stand-in for slab.CudaStepper: same interface, oracle compute."""

    def __init__(self, orc):
        self.orc = orc

    def tensor(self, block):
        return torch.from_numpy(block)  # shares memory with the numpy block

    def step_range(self, pre, post, z0, z1):
        self.orc.step_range(pre, post, z0, z1)
        self.orc.open_pass_range(post, z0, z1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, geom, steps, omega, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        f = random_block(np.random.default_rng(20240917), grid.size, np.float64)
        z0, z1 = slab.partition(nz, world)[rank]
        n = z1 - z0
        xp = nx + 2
        lo, hi = slab.exchange_flag_halos(flags[z0:z1], rank, world)
        want_lo, want_hi = slab.slab_halo_flags(flags, nx, ny, z0, z1)
        assert (lo == want_lo).all() and (hi == want_hi).all()
        fl = np.ones((n + 2, ny, xp), dtype=np.uint8)
        fl[1:-1, :, :nx], fl[0, :, :nx], fl[-1, :, :nx] = flags[z0:z1], lo, hi
        blocks = []
        for _ in range(2):
            blk = np.full((19, n + 2, ny, xp), np.nan)
            blk[:, 1:-1, :, :nx] = f.reshape(19, nz, ny, nx)[:, z0:z1]
            blocks.append(blk)
        runner = slab.DistSlab(OracleStepper(SlabOracle(nx, ny, n, xp, fl, omega, wall_u, inlet_u)),
                               n, rank, world)
        for r in runner.exchange(blocks[0]):
            r.wait()
        newest, _ = runner.run(blocks[0], blocks[1], steps)
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), newest[:, 1:-1, :, :nx])
        # whole-domain diagnostics: rank-ordered combine, identical on every rank
        mine = np.ascontiguousarray(newest[:, 1:-1, :, :nx])
        fluid = flags[z0:z1] == 0
        local = {"mass": float(mine.sum()), "px": float(rank), "py": 0.0, "pz": 0.0,
                 "kinetic_energy": 0.5 + rank, "max_u": 0.1 * (rank + 1), "nonfinite": 0.0,
                 "fluid_cells": float(fluid.sum())}
        total = slab.combine_diagnostics(local, rank, world)
        np.save(os.path.join(out_dir, f"diag{rank}.npy"),
                np.array([total[k] for k in slab.DIAG_KEYS]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel", "periodic"])
def test_two_rank_gloo_run_equals_single_domain(geom, tmp_path):
    world, steps, omega = 2, 5, 1.3
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    f = random_block(np.random.default_rng(20240917), grid.size, np.float64)
    want = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u).run(
        f.copy(), f.copy(), steps)
    mp.spawn(_worker, args=(world, _free_port(), geom, steps, omega, str(tmp_path)),
             nprocs=world, join=True)
    parts = [np.load(tmp_path / f"slab{r}.npy") for r in range(world)]
    got = np.concatenate(parts, axis=1)
    np.testing.assert_array_equal(got.reshape(19, -1), want)
    d0, d1 = np.load(tmp_path / "diag0.npy"), np.load(tmp_path / "diag1.npy")
    np.testing.assert_array_equal(d0, d1)                       # same bits on every rank
    diag = dict(zip(slab.DIAG_KEYS, d0))
    assert diag["mass"] == float(parts[0].sum()) + float(parts[1].sum())   # rank order
    assert diag["max_u"] == 0.2 and diag["px"] == 1.0 and diag["kinetic_energy"] == 2.0
    assert diag["fluid_cells"] == float((B.flatten_mask(grid) == 0).sum())


def test_single_rank_ring_closes_on_itself():
    grid, wall_u, inlet_u = geometries3d()["periodic"]
    nx, ny, nz = grid.shape
    flags = B.flatten_mask(grid).reshape(nz, ny, nx)
    f = random_block(np.random.default_rng(3), grid.size, np.float64)
    want = CpuOracle(nx, ny, nz, flags, 1.1).run(f.copy(), f.copy(), 3)
    lo, hi = slab.exchange_flag_halos(flags, 0, 1)
    fl = np.ones((nz + 2, ny, nx), dtype=np.uint8)
    fl[1:-1], fl[0], fl[-1] = flags, lo, hi
    blocks = [np.full((19, nz + 2, ny, nx), np.nan) for _ in range(2)]
    for blk in blocks:
        blk[:, 1:-1] = f.reshape(19, nz, ny, nx)
    runner = slab.DistSlab(OracleStepper(SlabOracle(nx, ny, nz, nx, fl, 1.1)), nz)
    runner.exchange(blocks[0])
    newest, _ = runner.run(blocks[0], blocks[1], 3)
    np.testing.assert_array_equal(newest[:, 1:-1].reshape(19, -1), want)


def _mismatch_worker(rank, world, port, same, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_16781_b200 import cases, engine
        from paper_2409_16781_b200.fields import Precision
        # a process group that serves a SWEEP: one simulation per rank, different physics
        spec = cases.CaseSpec("ldc", 8, 8, 8, re=50.0 if same else 50.0 + 25.0 * rank, u0=0.05)
        state = cases.init(spec, Precision.SINGLE)
        try:
            engine.run(state, engine.RunConfig(steps=1))
            outcome = "ran"
        except ValueError as exc:
            outcome = "ValueError: " + str(exc)
        except RuntimeError as exc:      # no CUDA device here: the decomposition itself was accepted
            outcome = "RuntimeError: " + str(exc)
        open(os.path.join(out_dir, f"out{rank}.txt"), "w").write(outcome)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the host-side guard without a GPU")
@pytest.mark.parametrize("same", [False, True])
def test_engine_run_decomposes_only_one_common_problem(same, tmp_path):
    """With a process group initialised engine.run treats the ranks' states as
    ONE z-decomposed domain - but only after checking that they ARE one (shape,
    step, physics, mask).  Ranks holding different problems (a sweep) all get a
    ValueError telling them to pass distributed=False; nobody hangs in a
    collective."""
    mp.spawn(_mismatch_worker, args=(2, _free_port(), same, str(tmp_path)), nprocs=2, join=True)
    outs = [open(tmp_path / f"out{r}.txt").read() for r in range(2)]
    if same:
        assert all(o.startswith("RuntimeError") for o in outs), outs   # reached the CUDA path
    else:
        assert all(o.startswith("ValueError") and "distributed=False" in o for o in outs), outs
