"""z-slab decomposition on the GPU: P logical slabs on ONE device (each
with its own plan, halo planes and halo flags, exchanging the 5 crossing
populations through mlb_halo_copy) must reproduce the single-domain run bit
for bit; so must the DistSlab driver with its boundary-first / interior
stream overlap."""

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision

from .helpers import geometries3d, random_block

pytestmark = pytest.mark.gpu


def single_domain(grid, prec, omega, wall_u, inlet_u, f, steps):
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = grid.shape
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), omega, wall_u,
                      inlet_u=inlet_u)
    a, b = plan.alloc(), plan.alloc()
    plan.upload(f, a)
    plan.upload(f, b)
    newest, _, _ = plan.run_steps(a, b, steps)
    out = np.empty_like(f)
    plan.download(newest, out)
    return out


def make_slabs(grid, prec, omega, wall_u, inlet_u, f, parts):
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = grid.shape
    flags = B.flatten_mask(grid).reshape(nz, ny, nx)
    dense = f.reshape(19, nz, ny, nx)
    slabs = []
    for (z0, z1) in slab.partition(nz, parts):
        lo, hi = slab.slab_halo_flags(flags, nx, ny, z0, z1)
        plan = KernelPlan(nx, ny, z1 - z0, Layout.ROW, prec, flags[z0:z1], omega, wall_u,
                          inlet_u=inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
        blocks = [plan.alloc(), plan.alloc()]
        part = np.ascontiguousarray(dense[:, z0:z1]).reshape(19, -1)
        for blk in blocks:
            blk.tensor.fill_(float("nan"))
            plan.upload(part, blk)
        slabs.append((plan, blocks, z0, z1))
    return slabs


def gather(slabs, which, like):
    parts = []
    for plan, blocks, z0, z1 in slabs:
        out = np.empty((19, (z1 - z0) * plan.ny * plan.nx), dtype=like.dtype)
        plan.download(blocks[which], out)
        parts.append(out.reshape(19, z1 - z0, plan.ny, plan.nx))
    return np.concatenate(parts, axis=1).reshape(19, -1)


@pytest.mark.parametrize("tag", ["f64", "f32"])
@pytest.mark.parametrize("parts", [1, 2, 3])
@pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel", "periodic"])
def test_logical_slabs_equal_single_domain_bitwise(geom, parts, tag, rng):
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = Precision.DOUBLE if tag == "f64" else Precision.SINGLE
    f = random_block(rng, grid.size, prec.storage)
    steps, omega = 5, 1.2
    want = single_domain(grid, prec, omega, wall_u, inlet_u, f, steps)
    slabs = make_slabs(grid, prec, omega, wall_u, inlet_u, f, parts)

    def exchange(which):
        for r, (plan, blocks, _, _) in enumerate(slabs):
            below = slabs[(r - 1) % parts]
            above = slabs[(r + 1) % parts]
            plan.halo_copy(blocks[which], below[1][which], face=0)
            plan.halo_copy(blocks[which], above[1][which], face=1)

    exchange(0)
    pre, post = 0, 1
    for _ in range(steps):
        for plan, blocks, z0, z1 in slabs:
            plan.step_range(blocks[pre], blocks[post], 0, z1 - z0)
            plan.open_pass_range(blocks[post], 0, z1 - z0)
        exchange(post)
        pre, post = post, pre
    np.testing.assert_array_equal(gather(slabs, pre, f), want)
    # and against the CPU oracle
    nx, ny, nz = grid.shape
    orc = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u)
    np.testing.assert_array_equal(want, orc.run(f.copy(), f.copy(), steps))


@pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel", "periodic"])
def test_distslab_overlap_path_single_rank(geom, rng):
    """DistSlab on CUDA with world = 1: boundary planes on the high-priority
    stream, interior on the main stream, ring closed on the slab itself."""
    from paper_2409_16781_b200 import slab
    grid, wall_u, inlet_u = geometries3d()[geom]
    f = random_block(rng, grid.size, np.float32)
    steps, omega = 6, 1.5
    want = single_domain(grid, Precision.SINGLE, omega, wall_u, inlet_u, f, steps)
    (plan, blocks, z0, z1), = make_slabs(grid, Precision.SINGLE, omega, wall_u, inlet_u, f, 1)
    runner = slab.DistSlab(slab.CudaStepper(plan), z1 - z0)
    assert runner.overlap
    runner.exchange(blocks[0])
    newest, _ = runner.run(blocks[0], blocks[1], steps)
    out = np.empty_like(f)
    plan.download(newest, out)
    np.testing.assert_array_equal(out, want)


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("tag", ["f64", "f32", "f16", "m2"])
@pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel", "periodic", "cavity16",
                                  "channel40", "open_chain", "open_unfusable"])
def test_peer_ring_single_rank(geom, tag, overlap, rng):
    """The fused exchange (PeerRing): the boundary-plane launches store the
    crossing populations into the ring neighbour's halo planes themselves.
    World = 1, so the neighbour is the slab's own block; strict and
    pass-through stores, fused and list-driven open-boundary pass."""
    from paper_2409_16781_b200 import slab
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE, "f16": Precision.MIXED1,
            "m2": Precision.MIXED2}[tag]
    f = random_block(rng, grid.size, prec.storage)
    steps, omega = 5, 1.4
    want = single_domain(grid, prec, omega, wall_u, inlet_u, f, steps)
    for passthrough in (False, True):
        (plan, blocks, z0, z1), = make_slabs(grid, prec, omega, wall_u, inlet_u, f, 1)
        if passthrough:
            try:
                plan.set_passthrough(True)
            except ValueError:
                continue  # chained outlets: the library refuses the mode
        ring = slab.PeerRing(plan, blocks)
        runner = slab.DistSlab(slab.CudaStepper(plan), z1 - z0, overlap=overlap, ring=ring)
        assert runner.overlap == (overlap and z1 - z0 >= 3)
        runner.exchange(blocks[0])
        newest, _ = runner.run(blocks[0], blocks[1], steps)
        runner.finish()
        out = np.empty_like(f)
        plan.download(newest, out)
        np.testing.assert_array_equal(out, want)
        # the halos of the newest block are what a plain halo copy would deliver
        got = newest.tensor.clone()
        plan.halo_copy(newest, newest, face=0)
        plan.halo_copy(newest, newest, face=1)
        import torch
        nx = plan.nx
        fluidish = torch.isfinite(got[:, :, :, :nx].float())
        assert torch.equal(got[:, :, :, :nx][fluidish], newest.tensor[:, :, :, :nx][fluidish])
        ring.close()


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("steps", [1, 2, 7])
@pytest.mark.parametrize("tag,variant", [("f32", 1008), ("f64", 1016), ("f16", 2008)])
@pytest.mark.parametrize("geom", ["cavity16", "periodic8", "porous", "channel40"])
def test_inplace_slab_single_rank(geom, tag, variant, steps, overlap, rng):
    """The in-place update on a z-slab (halo planes, peer ring closed on the
    slab's own block): the pull half stores its crossing results into the
    'neighbour's' boundary planes, the local half refills the halo planes."""
    from paper_2409_16781_b200 import slab
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE, "f16": Precision.MIXED1}[tag]
    f = random_block(rng, grid.size, prec.storage)
    omega = 1.4
    nx, ny, nz = grid.shape
    want = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u).run(
        f.copy(), f.copy(), steps)
    (plan, blocks, z0, z1), = make_slabs(grid, prec, omega, wall_u, inlet_u, f, 1)
    plan.set_variant(variant)
    blk = blocks[0]
    ring = slab.PeerRing(plan, [blk])
    runner = slab.DistSlab(slab.CudaStepper(plan), z1 - z0, overlap=overlap, ring=ring)
    runner.exchange(blk)
    runner.run_inplace(blk, steps)
    assert blk.repr == steps % 2
    runner.normalize(blk)
    out = np.empty_like(f)
    plan.download(blk, out)
    np.testing.assert_array_equal(out, want)
    # and on from the normalised state: halos were refilled
    runner.run_inplace(blk, 2)
    runner.normalize(blk)
    plan.download(blk, out)
    want2 = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u).run(
        want.copy(), want.copy(), 2)
    np.testing.assert_array_equal(out, want2)
    ring.close()


@pytest.mark.parametrize("tag", ["f32", "f64"])
@pytest.mark.parametrize("c_loop", [True, False])
def test_chained_outlets_with_boundary_and_interior_in_flight_together(tag, c_loop, rng):
    """An outlet cell whose source is itself an outlet cell makes the open-boundary
    pass gather-then-scatter through a scratch block (numpy evaluates the right-
    hand side first, engine.py:179-180).  In the z-slab schedule the pass runs on
    the boundary planes (high-priority stream) and on the interior (main stream)
    AT THE SAME TIME: each plane range must use its own part of the scratch.
    (Found by the fuzz suite at 4000 cases: the two launches shared it.)"""
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    prec = {"f32": Precision.SINGLE, "f64": Precision.DOUBLE}[tag]
    nx, ny, nz, steps = 96, 48, 24, 25
    grid = B.channel_mask(nx, ny, nz, B.sphere_cells(nx, ny, nz, 10, 30.0, 24.0, 12.0),
                          z_walls=False)
    grid[nx - 2, 1:-1, :] = B.OUTLET          # two outlet columns: x = nx-1 copies x = nx-2
    flags = B.flatten_mask(grid).reshape(nz, ny, nx)
    f = random_block(rng, grid.size, prec.storage)
    want = CpuOracle(nx, ny, nz, flags, 1.2, (0.0, 0.0, 0.0), 0.05, threads=8).run(
        f.copy(), f.copy(), steps)
    lo, hi = slab.slab_halo_flags(flags, nx, ny, 0, nz)
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, flags, 1.2, (0.0, 0.0, 0.0), inlet_u=0.05,
                      halo_lo=lo, halo_hi=hi, slab=True)
    with pytest.raises(ValueError, match="outlet"):
        plan.set_passthrough(True)            # chained outlets: strict stores, list-driven pass
    for rep in range(3):                      # a race shows up some of the time
        a, b = plan.alloc(), plan.alloc()
        for blk in (a, b):
            blk.tensor.fill_(float("nan"))
            plan.upload(f, blk)
        ring = slab.PeerRing(plan, [a, b])
        runner = slab.DistSlab(slab.CudaStepper(plan), nz, overlap=True, ring=ring, c_loop=c_loop)
        runner.exchange(a)
        newest, _ = runner.run(a, b, steps)
        runner.finish()
        got = np.empty_like(f)
        plan.download(newest, got)
        ring.close()
        np.testing.assert_array_equal(got, want)
