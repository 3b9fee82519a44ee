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
  2. the exchange as soon as (1) is done;
  3. the interior planes on the main stream, concurrently with (2);
  4. join, swap.
The data path has no collective - only the two neighbour exchanges.

Two transports for (2):
* `PeerRing` (the product path on one NVSwitch box): every rank maps its ring
  neighbours' population blocks (CUDA IPC) and the boundary-plane launch of (1)
  stores the crossing populations straight into the neighbour's halo planes
  from inside the fused kernel - no pack buffer, no copy kernel, no NCCL call
  on the data path.  Ordering between ranks is a pair of monotone step
  counters per rank in device memory: after its boundary launches of step t a
  rank posts t into both neighbours' counters; before its boundary launches of
  step t it makes its stream wait (stream memory operation, no host sync)
  until both neighbours have posted t-1 - which says both that the halos it is
  about to read are complete and that the halos it is about to overwrite have
  been read.
* torch.distributed send/recv (NCCL over NVLink on GPUs, gloo on CPU): the
  portable fallback, and what the CPU tests drive.

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


class PeerRing:
    """The ring neighbours' blocks and step counters, mapped into this process.

    `blocks` are this rank's population blocks (DeviceFields of `plan`): two
    for the two-buffer update, one for the in-place update;
    every rank passes its own and learns the others' through one object
    all-gather of CUDA IPC handles (64 bytes each) - control plane only.
    With world == 1 the ring closes on the rank's own blocks.
    """

    SLOT_FROM_BELOW, SLOT_FROM_ABOVE = 0, 128  # byte offsets inside the signal block

    def __init__(self, plan, blocks, rank=0, world=1, group=None, wait_mode=0):
        import ctypes
        from . import _cabi
        self.plan, self.blocks = plan, list(blocks)
        self.rank, self.world, self.group = rank, world, group
        self.wait_mode = int(wait_mode)
        self._lib = lib = _cabi.lib()
        self._ct = ctypes
        self._check = _cabi.check
        self.t = 0           # steps posted so far
        self._opened = {}    # handle bytes -> mapped base address
        dev = plan.device.index
        sig = ctypes.c_void_p()
        _cabi.check(lib.mlb_signal_create(dev, ctypes.byref(sig)))
        self.sig = sig.value
        below, above = ring_neighbours(rank, world)
        if world == 1:
            mine = {"nz": plan.nz, "blocks": [b.tensor.data_ptr() for b in self.blocks],
                    "sig": self.sig}
            self.below = self.above = mine
            return
        import torch.distributed as dist
        # every rank reaches the all-gather, also one whose export failed (its
        # card then carries the error and every rank raises the same way)
        try:
            card = {"nz": plan.nz,
                    "blocks": [self._export(b.tensor.data_ptr()) for b in self.blocks],
                    "sig": self._export(self.sig)}
        except (RuntimeError, ValueError) as exc:
            card = {"error": f"rank {rank}: {exc}"}
        cards = [None] * world
        dist.all_gather_object(cards, card, group=group)
        errors = [c["error"] for c in cards if "error" in c]
        if errors:
            lib.mlb_signal_destroy(ctypes.c_void_p(self.sig))
            self.sig = None
            raise RuntimeError("peer ring: " + "; ".join(errors))
        self.below = self._map(cards[below])
        self.above = self.below if above == below else self._map(cards[above])

    def _export(self, ptr):
        ct = self._ct
        handle = ct.create_string_buffer(64)
        off = ct.c_int64()
        self._check(self._lib.mlb_ipc_export(ct.c_void_p(ptr), handle, ct.byref(off)))
        return handle.raw, off.value

    def _open(self, handle, off):
        ct = self._ct
        if handle not in self._opened:
            base = ct.c_void_p()
            self._check(self._lib.mlb_ipc_open(self.plan.device.index, handle, ct.byref(base)))
            self._opened[handle] = base.value
        return self._opened[handle] + off

    def _map(self, card):
        return {"nz": card["nz"], "blocks": [self._open(*h) for h in card["blocks"]],
                "sig": self._open(*card["sig"])}

    def index(self, block):
        for k, b in enumerate(self.blocks):
            if b is block:
                return k
        raise ValueError("block is not one of the ring's population blocks")

    def targets(self, k):
        """((below ptr, nz), (above ptr, nz)) for pushes out of local block k."""
        return ((self.below["blocks"][k], self.below["nz"]),
                (self.above["blocks"][k], self.above["nz"]))

    def c_ring(self, first, overlap):
        """This rank's view of the ring as the library's `mlb_ring`, for the
        one-call loops (mlb_slab_run_steps*): `first` is the local block that
        plays d_a (index 0 of the struct's block arrays)."""
        from . import _cabi
        r = _cabi.Ring()
        order = [first] + [k for k in range(len(self.blocks)) if k != first]
        for j, k in enumerate(order):
            r.below[j] = self.below["blocks"][k]
            r.above[j] = self.above["blocks"][k]
        r.nz_below, r.nz_above = self.below["nz"], self.above["nz"]
        # I am the slab ABOVE my below-neighbour, and BELOW my above-neighbour
        r.post_below = self.below["sig"] + self.SLOT_FROM_ABOVE
        r.post_above = self.above["sig"] + self.SLOT_FROM_BELOW
        r.wait_below = self.sig + self.SLOT_FROM_BELOW
        r.wait_above = self.sig + self.SLOT_FROM_ABOVE
        r.t, r.wait_mode, r.overlap = self.t, self.wait_mode, int(bool(overlap))
        return r

    def _stream(self):
        return self._ct.c_void_p(torch.cuda.current_stream(self.plan.device).cuda_stream)

    def wait(self, value):
        """Current stream waits until both neighbours have posted `value`."""
        for off in (self.SLOT_FROM_BELOW, self.SLOT_FROM_ABOVE):
            self._check(self._lib.mlb_signal_wait(self._ct.c_void_p(self.sig + off), value,
                                                  self.wait_mode, self._stream()))

    def post(self, value):
        """After everything enqueued so far on the current stream: tell both
        neighbours this rank's boundary planes of step `value` are done (its
        pushes into their halos have landed, their halos in the other block
        have been read)."""
        # I am the slab ABOVE my below-neighbour, and BELOW my above-neighbour
        self._check(self._lib.mlb_signal_post(
            self._ct.c_void_p(self.below["sig"] + self.SLOT_FROM_ABOVE), value, self._stream()))
        self._check(self._lib.mlb_signal_post(
            self._ct.c_void_p(self.above["sig"] + self.SLOT_FROM_BELOW), value, self._stream()))
        self.t = value

    def barrier(self):
        torch.cuda.synchronize(self.plan.device)
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    def exchange(self, k):
        """Fill the neighbours' halo planes of block k from this rank's
        boundary planes (setup; the per-step exchange is fused into the
        kernel).  Collective: returns when every rank's halos are filled."""
        self.barrier()
        (bp, bn), (ap, an) = self.targets(k)
        self.plan.halo_push(self.blocks[k], ap, an, face=0)
        self.plan.halo_push(self.blocks[k], bp, bn, face=1)
        self.barrier()

    def close(self):
        if getattr(self, "sig", None) is None:
            return
        self.barrier()   # nobody is still storing into a mapping we are about to drop
        for base in self._opened.values():
            self._lib.mlb_ipc_close(self._ct.c_void_p(base))
        self._opened = {}
        self.barrier()
        self._lib.mlb_signal_destroy(self._ct.c_void_p(self.sig))
        self.sig = None


class DistSlab:
    """One rank's slab of a z-decomposed run over torch.distributed.

    `stepper` advances plane ranges of this rank's slab; `pre` / `post` are
    its population blocks, anything `stepper.tensor()` turns into a torch
    tensor of shape (19, nz+2, ny, xp).  With world == 1 the ring closes on
    the slab itself and the exchange is a local copy.
    """

    def __init__(self, stepper, nz_local, rank=0, world=1, group=None,
                 overlap=True, ring=None, force_dist=False, c_loop=True):
        self.stepper = stepper
        # with a peer ring, `run` / `run_inplace` hand the whole loop to the
        # library (mlb_slab_run_steps*: the same schedule as `step`, no Python
        # between steps); c_loop=False keeps the step-by-step Python schedule
        self.c_loop = bool(c_loop)
        self.host_us_per_step = None   # of the last one-call loop
        self.nz = int(nz_local)
        self.rank, self.world, self.group = rank, world, group
        self.below, self.above = ring_neighbours(rank, world)
        self.cuda = isinstance(stepper, CudaStepper)
        self.overlap = bool(overlap) and self.cuda and self.nz >= 3
        self.ring = ring  # PeerRing: fused peer-store exchange instead of send/recv
        # world == 1 normally closes the ring with local copies; force_dist sends
        # the planes through torch.distributed to this same rank instead (lets a
        # one-GPU box exercise the NCCL send/recv path)
        self.force_dist = bool(force_dist)
        if ring is not None and not self.cuda:
            raise ValueError("the peer-memory ring needs the CUDA stepper")

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
        if self.ring is not None:
            self.ring.exchange(self.ring.index(block))
            return []
        t = self.stepper.tensor(block)
        sends, recvs = self._ops(t)
        if self.world == 1 and not self.force_dist:
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
        if self.ring is not None:
            return self._step_ring(pre, post)
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

    def _step_ring(self, pre, post):
        """One step with the exchange fused into the boundary-plane launches
        (PeerRing).  Step t's boundary launches wait for both neighbours'
        post of t-1, push into the neighbours' halos of the same-index block,
        and post t."""
        st, nz, ring = self.stepper, self.nz, self.ring
        plan = st.plan
        below, above = ring.targets(ring.index(post))
        t = ring.t + 1
        if not self.overlap:
            ring.wait(t - 1)
            plan.step_push_range(pre, post, 0, nz, below, above)
            ring.post(t)
            return
        main = torch.cuda.current_stream(st.device)
        ready = torch.cuda.Event()
        ready.record(main)
        st.hi.wait_event(ready)
        with torch.cuda.stream(st.hi):
            ring.wait(t - 1)
            plan.step_push_range(pre, post, 0, 1, below, None)
            plan.step_push_range(pre, post, nz - 1, nz, None, above)
            ring.post(t)
        st.step_range(pre, post, 1, nz - 1)  # interior: no halo, no neighbour involved
        done = torch.cuda.Event()
        done.record(st.hi)
        main.wait_event(done)

    # -- the in-place update over slabs (one block per rank, PeerRing) ----------
    def step_inplace(self, f):
        """One in-place step of this slab (mlb_step_inplace_range): the pull
        half writes its results for the crossing directions into the
        neighbours' boundary planes, the local half refills the neighbours'
        halo planes.  Same boundary-first schedule and the same step counters
        as the two-buffer step."""
        st, nz, ring = self.stepper, self.nz, self.ring
        if ring is None:
            raise ValueError("the in-place slab step needs the peer-memory ring")
        plan = st.plan
        below, above = ring.targets(ring.index(f))
        t = ring.t + 1
        if not self.overlap:
            ring.wait(t - 1)
            plan.step_inplace_range(f, 0, nz, below, above)
            ring.post(t)
        else:
            main = torch.cuda.current_stream(st.device)
            ready = torch.cuda.Event()
            ready.record(main)
            st.hi.wait_event(ready)
            with torch.cuda.stream(st.hi):
                ring.wait(t - 1)
                plan.step_inplace_range(f, 0, 1, below, above)
                plan.step_inplace_range(f, nz - 1, nz, below, above)
                ring.post(t)
            plan.step_inplace_range(f, 1, nz - 1, below, above)
            done = torch.cuda.Event()
            done.record(st.hi)
            main.wait_event(done)
        f.repr ^= 1

    def _loop_args(self):
        import ctypes
        st = self.stepper
        main = ctypes.c_void_p(torch.cuda.current_stream(st.device).cuda_stream)
        hi = ctypes.c_void_p(st.hi.cuda_stream)
        return ctypes, main, hi, ctypes.c_double(0.0)

    def run_inplace(self, f, nsteps):
        if self.ring is None or not self.c_loop:
            for _ in range(nsteps):
                self.step_inplace(f)
            return f
        from . import _cabi
        ct, main, hi, us = self._loop_args()
        ring = self.ring.c_ring(self.ring.index(f), self.overlap)
        r = ct.c_int(f.repr)
        _cabi.check(_cabi.lib().mlb_slab_run_steps_inplace(
            self.stepper.plan._plan, f.ptr, int(nsteps), ct.byref(r), ct.byref(ring), main, hi,
            ct.byref(us)))
        f.repr, self.ring.t, self.host_us_per_step = r.value, int(ring.t), us.value
        return f

    def normalize(self, f):
        """Bring an in-place slab back to the normal representation (a no-op
        after an even number of steps).  Collective.

        In place the neighbours' next pull half writes into THIS rank's
        boundary planes, so whatever reads the block afterwards (probe,
        diagnostics, download) must be finished on every rank before anyone
        steps on: call `fence()` between the reads and the next step."""
        ring = self.ring
        ring.barrier()
        if f.repr == 1:
            k = ring.index(f)
            below, above = ring.targets(k)
            self.stepper.plan.inplace_swap_slab(f, above)
            f.repr = 0
            ring.barrier()          # every slab normal before any halo is refilled
            ring.exchange(k)
        ring.barrier()

    def fence(self):
        """Device synchronisation + barrier over the ring's ranks."""
        self.ring.barrier()

    def finish(self):
        """After the last step, before anyone reads halos or frees blocks:
        every rank's pushes have landed."""
        if self.ring is not None:
            self.ring.barrier()

    def run(self, a, b, nsteps):
        """`nsteps` steps alternating a -> b -> a; returns (newest, other)."""
        if self.ring is not None and self.c_loop and self.cuda:
            from . import _cabi
            ct, main, hi, us = self._loop_args()
            ring = self.ring.c_ring(self.ring.index(a), self.overlap)
            _cabi.check(_cabi.lib().mlb_slab_run_steps(
                self.stepper.plan._plan, a.ptr, b.ptr, int(nsteps), ct.byref(ring), main, hi,
                ct.byref(us)))
            self.ring.t, self.host_us_per_step = int(ring.t), us.value
            return (a, b) if nsteps % 2 == 0 else (b, a)
        import time
        pre, post = a, b
        t0 = time.perf_counter()
        for k in range(nsteps):
            self.step(pre, post)
            pre, post = post, pre
            if k < 32:      # host time per step, before the launch queue can fill
                self.host_us_per_step = (time.perf_counter() - t0) / (k + 1) * 1e6
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


def _agree(ok, world, group, device):
    """Every rank takes the same branch: True only if all ranks say so."""
    if world == 1:
        return bool(ok)
    import torch.distributed as dist
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


def halo_planes(block, nz):
    """The ten halo planes the exchange fills, stacked (for comparisons)."""
    t = block.tensor
    return torch.stack([t[q, 0] for q in UP] + [t[q, nz + 1] for q in DOWN])


def halos_match_send_recv(plan, block, rank, world, group=None):
    """Cross-check of the fused exchange on live data: are the halo planes
    `block` holds exactly the planes a send/recv exchange delivers?  Runs
    that exchange (which rewrites the same planes with the same data when
    the answer is yes).  Collective; needs a backend that moves CUDA tensors
    point to point (NCCL) - returns True untested otherwise."""
    if world == 1:
        return True
    import torch.distributed as dist
    if dist.get_backend(group) != "nccl":
        return True
    got = halo_planes(block, plan.nz).clone()
    for r in DistSlab(CudaStepper(plan), plan.nz, rank, world, group).exchange(block):
        r.wait()
    torch.cuda.synchronize(plan.device)
    return _agree(torch.equal(got, halo_planes(block, plan.nz)), world, group, plan.device)


def open_runner(plan, a, b, rank=0, world=1, group=None, transport="peer", overlap=True):
    """A DistSlab for this rank's slab with its halos filled, and the name
    of the transport it uses.

    transport "peer": the fused peer-store exchange (PeerRing) when every
    rank can map its neighbours and the ring delivers exactly the planes
    send/recv delivers; otherwise - and with transport "nccl" - the
    send/recv exchange, the returned name saying why.  Collective."""
    dev = plan.device
    why = None
    if transport == "peer":
        ring, err = None, None
        try:
            ring = PeerRing(plan, [a, b], rank, world, group)
        except Exception as exc:  # cudaIpc* refused (allocator, no P2P, ...)
            err = f"{type(exc).__name__}: {exc}"
        if _agree(ring is not None, world, group, dev):
            runner = DistSlab(CudaStepper(plan), plan.nz, rank, world, group,
                              overlap=overlap, ring=ring)
            runner.exchange(a)
            if halos_match_send_recv(plan, a, rank, world, group):
                return runner, "peer"
            why = "pre-flight mismatch against send/recv"
            ring.close()
        else:
            why = err or "a peer rank could not map the ring"
            if ring is not None:
                ring.close()
    runner = DistSlab(CudaStepper(plan), plan.nz, rank, world, group, overlap=overlap)
    for r in runner.exchange(a):
        r.wait()
    return runner, "nccl" if why is None else f"nccl (peer ring unavailable: {why})"


def open_inplace_runner(plan, f, rank=0, world=1, group=None, overlap=True):
    """A DistSlab that advances ONE block per rank in place.  The in-place
    exchange writes into the neighbours' boundary planes, so it exists over
    peer memory only: if some rank cannot map its neighbours every rank
    raises.  Collective."""
    ring, err = None, None
    try:
        ring = PeerRing(plan, [f], rank, world, group)
    except Exception as exc:
        err = f"{type(exc).__name__}: {exc}"
    if not _agree(ring is not None, world, group, plan.device):
        if ring is not None:
            ring.close()
        raise RuntimeError("the in-place update over z-slabs needs peer memory between the "
                           "ranks (CUDA IPC): " + (err or "a peer rank could not map the ring"))
    # Can every rank's slab be served in place (pack kernel, outlet cells inside their
    # packs)?  The geometry differs from slab to slab, so one rank alone might refuse at
    # its first launch while its neighbours wait for its step counter: ask all, agree.
    below, above = ring.targets(0)
    try:
        plan.step_inplace_range(f, 0, 0, below, above)     # empty plane range: the checks only
        why = None
    except ValueError as exc:
        why = str(exc)
    if not _agree(why is None, world, group, plan.device):
        ring.close()
        raise ValueError("the in-place update cannot serve the slab of some rank"
                         + (f" (this rank: {why})" if why else ""))
    runner = DistSlab(CudaStepper(plan), plan.nz, rank, world, group, overlap=overlap, ring=ring)
    runner.exchange(f)
    return runner


DIAG_KEYS = ("mass", "px", "py", "pz", "kinetic_energy", "max_u", "nonfinite", "fluid_cells")


def combine_diagnostics(local, rank=0, world=1, group=None):
    """Whole-domain diagnostics from every slab's `KernelPlan.diagnostics()`.

    The per-slab values are deterministic device reductions; they are
    gathered (8 doubles per rank, control plane) and combined on every rank
    in RANK ORDER - sums left to right, max |u| by max - so the result is
    bitwise reproducible and identical on all ranks (no floating-point
    all-reduce whose order the library picks)."""
    mine = [float(local[k]) for k in DIAG_KEYS]
    if world == 1:
        rows = [mine]
    else:
        import torch.distributed as dist
        rows = [None] * world
        dist.all_gather_object(rows, mine, group=group)
    out = dict(zip(DIAG_KEYS, rows[0]))
    for row in rows[1:]:
        for k, v in zip(DIAG_KEYS, row):
            out[k] = max(out[k], v) if k == "max_u" else out[k] + v
    return out


__all__ = ["combine_diagnostics", "DIAG_KEYS", "open_runner", "open_inplace_runner", "halos_match_send_recv",
           "halo_planes", "partition", "ring_neighbours", "slab_halo_flags", "CudaStepper",
           "PeerRing", "DistSlab", "exchange_flag_halos", "Q"]
