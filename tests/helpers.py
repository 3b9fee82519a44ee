"""Shared test helpers: geometries, random fields, the z-projection bridge."""

import numpy as np

from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import lattice as L


def geometries3d():
    """3-D counterparts of the reference's kernel-test geometries
    (pkg/tests/test_kernels.py:25-33), small and ragged on purpose (no
    extent is a multiple of the 128-byte line)."""
    cavity = B.cavity_mask(9, 7, 5)
    cavity[4, 3, 2] = B.SOLID  # interior obstacle
    channel = B.channel_mask(14, 9, 8, B.sphere_cells(14, 9, 8, 4, 5.0, 4.0, 3.5))
    duct = B.channel_mask(12, 8, 6, B.cylinder_cells(12, 8, 6, 4, 4.0, 3.5),
                          z_walls=False)
    periodic = B.open_mask(6, 5, 4)
    # row lengths that are multiples of the 16-byte pack: these exercise the
    # vectorised kernel (several packs per row, walls inside and between packs)
    cavity16 = B.cavity_mask(16, 9, 7)
    cavity16[5:8, 3:5, 2:4] = B.SOLID
    cavity16[11, 6, 4] = B.SOLID
    channel40 = B.channel_mask(40, 10, 6, B.sphere_cells(40, 10, 6, 4, 9.0, 4.5, 2.5))
    periodic8 = B.open_mask(8, 5, 4)
    periodic8[3, 2, 1] = B.SOLID
    periodic8[4, 2, 1] = B.MOVING_WALL
    wide = B.open_mask(72, 4, 3)
    # open-boundary cells in arbitrary places (the reference's pass works on
    # index lists, engine.py:161-174): an inlet column mid-domain, a CHAIN of
    # outlet cells (each copying its west neighbour's pre-pass value), walls
    open_chain = B.open_mask(16, 6, 4)
    open_chain[5, 1:5, :] = B.INLET
    open_chain[13:16, 2:4, 1:3] = B.OUTLET
    open_chain[9, 3, 2] = B.SOLID
    open_chain[:, 0, :] = B.SOLID
    # an outlet cell that starts a 16-byte pack (x % 4 == 0): cannot ride in
    # the pack kernel, must fall back to the list-driven pass
    open_unfusable = open_chain.copy()
    open_unfusable[8, 4, 1:3] = B.OUTLET
    # random porous medium with moving grains: far more than 254 distinct
    # wall-link patterns, so the plan's pattern dictionary overflows and the
    # escape path (full-width class words) is exercised
    prng = np.random.default_rng(7)
    porous = B.open_mask(24, 10, 8)
    u = prng.random(porous.shape)
    porous[u < 0.25] = B.SOLID
    porous[u > 0.9] = B.MOVING_WALL
    return {"cavity": (cavity, (0.08, 0.0, 0.0), 0.0),
            "porous": (porous, (0.03, -0.02, 0.04), 0.0),
            "cavity16": (cavity16, (0.05, 0.0, -0.03), 0.0),
            "channel40": (channel40, (0.0, 0.0, 0.0), 0.06),
            "periodic8": (periodic8, (0.02, 0.03, -0.04), 0.0),
            "wide": (wide, (0.0, 0.0, 0.0), 0.0),
            "open_chain": (open_chain, (0.0, 0.0, 0.0), 0.04),
            "open_unfusable": (open_unfusable, (0.0, 0.0, 0.0), 0.04),
            "cavity_oblique_lid": (cavity, (0.05, 0.0, -0.03), 0.0),
            "channel": (channel, (0.0, 0.0, 0.0), 0.07),
            "duct": (duct, (0.0, 0.0, 0.0), 0.05),
            "periodic": (periodic, (0.0, 0.0, 0.0), 0.0)}


def random_block(rng, n, dtype):
    """Populations ~ U(0.02, 1) as the reference's tests draw them
    (test_kernels.py:19-22)."""
    return np.ascontiguousarray(
        rng.uniform(0.02, 1.0, size=(19, n)).astype(dtype))


def lift_2d(f2, nz):
    """Lift a D2Q9 block (9, ny*nx) to a z-symmetric, z-invariant D3Q19
    block (19, nz*ny*nx) whose sum over c_z is f2 exactly: each 2-D
    population is split over its c_z group in proportion to the lattice
    weights (dyadic fractions, so the split is exact in floating point)."""
    n2 = f2.shape[1]
    f3 = np.zeros((19, nz, n2), dtype=f2.dtype)
    for k in range(9):
        grp = L.PROJECT_2D[k]
        wsum = L.W[grp].sum()
        for i in grp:
            f3[i] = (f2.dtype.type(L.W[i] / wsum) * f2[k])[None, :]
    return np.ascontiguousarray(f3.reshape(19, nz * n2))


def project_2d(f3, nz):
    """Sum a D3Q19 block over c_z: (nz, 9, ny*nx) float64."""
    f3 = np.asarray(f3, dtype=np.float64).reshape(19, nz, -1)
    out = np.zeros((nz, 9, f3.shape[2]))
    for k in range(9):
        for i in L.PROJECT_2D[k]:
            out[:, k] += f3[i]
    return out


def extrude_mask(mask2_flat, nx, ny, nz):
    """(ny*nx,) ROW-ordered 2-D flags -> dense [nz][ny][nx] flags."""
    m = np.asarray(mask2_flat, dtype=np.uint8).reshape(ny, nx)
    return np.ascontiguousarray(np.broadcast_to(m[None], (nz, ny, nx))).reshape(-1)


def to_xyzq(block, nx, ny, nz):
    """(19, N) block -> (nx, ny, nz, 19) float64 array for the naive oracle."""
    return np.ascontiguousarray(
        np.asarray(block, dtype=np.float64).reshape(19, nz, ny, nx).transpose(3, 2, 1, 0))


def from_xyzq(a):
    nx, ny, nz, _ = a.shape
    return np.ascontiguousarray(a.transpose(3, 2, 1, 0).reshape(19, nz * ny * nx))


def init_ranks(rank, world, port):
    """Process-group + device setup of a multi-process GPU test.  On a box with
    at least `world` GPUs every rank takes its own device and the control plane
    is NCCL - the exchange then really crosses NVLink; on a smaller box all
    ranks share device 0 over a gloo control plane (separate CUDA contexts,
    real IPC mappings, same protocol).  Returns (device index, the device
    argument for slab.exchange_flag_halos: None = host tensors)."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if torch.cuda.device_count() >= world and os.environ.get("MLB_TEST_SHARE_GPU") != "1":
        dev = rank
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
        return dev, torch.device("cuda", dev)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return 0, None
