"""z-slab domain decomposition: one slab per GPU, 5-population halos.

The reference is single-address-space; what it does prove is
that the update is partition-independent - each destination cell is written
exactly once from the read-only pre buffer (kernels.py:3-8), and tiling or
thread count never change a bit (test_kernels.py:107-126).  Slab
decomposition leans on exactly that property: rank r owns global planes
[z0, z1) plus one halo plane either side inside the same padded block, the
fused kernel pulls across the z faces from the halos without a branch, and
after every step only the populations that cross a face are exchanged with
the ring neighbours:

    plane lz = nz-1, c_z = +1 set {9, 11, 12, 15, 16}  ->  upper neighbour's halo lz = -1
    plane lz = 0,    c_z = -1 set {10, 13, 14, 17, 18}  ->  lower neighbour's halo lz = nz

(5 of 19 populations per face; each plane is one contiguous run of the SoA
layout, so there is no pack kernel).  The ring is periodic in z, as the
reference's wrap is (kernels.py:84-86); for a cavity or a walled channel
the wrap link carries data nobody reads, one code path either way.

Per step on each rank (DistSlab.step):
  1. boundary planes lz = 0 and lz = nz-1 (+ their open-boundary cells) on a
     high-priority stream;
  2. the exchange (NCCL send/recv over NVLink via torch.distributed) as soon
     as (1) is done;
  3. the interior planes on the main stream, concurrently with (2);
  4. join, swap.
The data path has no collective - only the two neighbour exchanges.

`DistSlab` is written against a small "stepper" interface so the same
driver code runs under `gloo` on CPU tensors in the tests (with the CPU
oracle as the stepper) and under `nccl` on the GPU (CudaStepper).
"""

import numpy as np
import torch

from .lattice import DOWN, UP, Q


def partition(nz, world):
    """Global planes [z0, z1) of each rank: as equal as possible, the first
    nz % world ranks get one extra plane."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} planes over {world} slabs")
    base, rem = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((z, z + n))
        z += n
    return out


def ring_neighbours(rank, world):
    """(below, above): the ranks owning the planes under z0 and over z1-1."""
    return (rank - 1) % world, (rank + 1) % world


def slab_halo_flags(flags_global, nx, ny, z0, z1):
    """The two halo flag planes of slab [z0, z1) cut from a dense global
    [nz][ny][nx] flag array (periodic in z)."""
    g = np.asarray(flags_global, dtype=np.uint8).reshape(-1, ny, nx)
    nz = g.shape[0]
    return g[(z0 - 1) % nz].copy(), g[z1 % nz].copy()


class CudaStepper:
    """The CUDA path behind the stepper interface DistSlab drives."""

    def __init__(self, plan):
        self.plan = plan
        self.device = plan.device
        self.hi = torch.cuda.Stream(self.device, priority=-1)

    def alloc(self):
        return self.plan.alloc()

    def tensor(self, field):
        return field.tensor

    def step_range(self, pre, post, z0, z1):
        self.plan.step_open_range(pre, post, z0, z1)


class DistSlab:
    """One rank's slab of a z-decomposed run over torch.distributed.

    `stepper` advances plane ranges of this rank's slab; `pre` / `post` are
    its population blocks, anything `stepper.tensor()` turns into a torch
    tensor of shape (19, nz+2, ny, xp).  With world == 1 the ring closes on
    the slab itself and the exchange is a local copy.
    """

    def __init__(self, stepper, nz_local, rank=0, world=1, group=None,
                 overlap=True):
        self.stepper = stepper
        self.nz = int(nz_local)
        self.rank, self.world, self.group = rank, world, group
        self.below, self.above = ring_neighbours(rank, world)
        self.cuda = isinstance(stepper, CudaStepper)
        self.overlap = bool(overlap) and self.cuda and self.nz >= 3

    # -- halo exchange -----------------------------------------------------
    def _ops(self, t):
        """(send views, recv views) as lists of (tensor, peer)."""
        nz = self.nz
        sends = [(t[q, nz], self.above) for q in UP] \
            + [(t[q, 1], self.below) for q in DOWN]
        recvs = [(t[q, 0], self.below) for q in UP] \
            + [(t[q, nz + 1], self.above) for q in DOWN]
        return sends, recvs

    def exchange(self, block):
        """Fill both halo planes of `block` from the ring neighbours."""
        t = self.stepper.tensor(block)
        sends, recvs = self._ops(t)
        if self.world == 1:
            for (src, _), (dst, _) in zip(sends, recvs):
                dst.copy_(src)
            return []
        import torch.distributed as dist
        # with two ranks both neighbours are the same peer: messages between
        # a pair match in posting order, and both sides post the UP set
        # first, then the DOWN set
        ops = []
        for (src, peer) in sends:
            ops.append(dist.P2POp(dist.isend, src, peer, self.group))
        for (dst, peer) in recvs:
            ops.append(dist.P2POp(dist.irecv, dst, peer, self.group))
        return dist.batch_isend_irecv(ops)

    # -- one time step -----------------------------------------------------
    def step(self, pre, post):
        """Advance this slab one step (fused update + open-boundary pass on
        every plane, then the halo exchange of `post`).  Returns when the
        work is enqueued (CUDA) or done (CPU); the caller swaps."""
        st, nz = self.stepper, self.nz
        if not self.overlap:
            st.step_range(pre, post, 0, nz)
            for r in self.exchange(post):
                r.wait()
            return
        main = torch.cuda.current_stream(st.device)
        ready = torch.cuda.Event()
        ready.record(main)            # everything before this step (incl. last exchange)
        st.hi.wait_event(ready)
        with torch.cuda.stream(st.hi):
            st.step_range(pre, post, 0, 1)
            st.step_range(pre, post, nz - 1, nz)
            reqs = self.exchange(post)  # NCCL orders itself after the hi stream
        st.step_range(pre, post, 1, nz - 1)  # interior, concurrent with the exchange
        with torch.cuda.stream(st.hi):
            for r in reqs:
                r.wait()
        done = torch.cuda.Event()
        done.record(st.hi)
        main.wait_event(done)

    def run(self, a, b, nsteps):
        """`nsteps` steps alternating a -> b -> a; returns (newest, other)."""
        pre, post = a, b
        for _ in range(nsteps):
            self.step(pre, post)
            pre, post = post, pre
        return pre, post


def exchange_flag_halos(flags_slab, rank, world, group=None, device=None):
    """Once at setup: the flag planes of the ring neighbours.

    `flags_slab` is this rank's dense [nz][ny][nx] uint8 block.  Returns
    (halo_lo, halo_hi) as (ny, nx) uint8 arrays: the top plane of the slab
    below and the bottom plane of the slab above.
    """
    f = np.ascontiguousarray(flags_slab, dtype=np.uint8)
    if world == 1:
        return f[-1].copy(), f[0].copy()
    import torch.distributed as dist
    below, above = ring_neighbours(rank, world)
    dev = device if device is not None else "cpu"
    top = torch.from_numpy(f[-1].copy()).to(dev)
    bottom = torch.from_numpy(f[0].copy()).to(dev)
    lo = torch.empty_like(top)
    hi = torch.empty_like(bottom)
    ops = [dist.P2POp(dist.isend, top, above, group),
           dist.P2POp(dist.isend, bottom, below, group),
           dist.P2POp(dist.irecv, lo, below, group),
           dist.P2POp(dist.irecv, hi, above, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    if dev != "cpu":
        torch.cuda.synchronize()
    return lo.cpu().numpy(), hi.cpu().numpy()


__all__ = ["partition", "ring_neighbours", "slab_halo_flags", "CudaStepper",
           "DistSlab", "exchange_flag_halos", "Q"]
