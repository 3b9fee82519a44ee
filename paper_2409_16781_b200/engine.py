"""Time stepping and run orchestration on the CUDA path.

Host-side mirror of /root/reference/pkg/src/lb2d/engine.py: `Schedule`
(:36-60), `RunConfig` (:63-81), `SimState` (:84-125),
`state_from_macroscopic` (:128-153), `build_plan` (:183-190), `step`
(:193-205), `run` -> `RunStats` (:208-275).  Same names, argument meaning
and error behaviour, one more dimension.  The reference's driver code keeps
working against host `SimState`s; what changes is where a step executes:

* the state's host arrays (dense `(19, N)` blocks, x fastest) stay the
  user-visible truth, exactly as in the reference;
* `run` uploads them to the padded device layout, advances on the GPU
  through the C ABI (fused kernel, open-boundary pass, swap - the
  reference's timed loop body, engine.py:244-249), fires the same hooks at
  the same cadence with the host arrays synchronised first, and downloads
  at the end.  `RunStats.seconds` is device time of the update loop from
  CUDA events (the reference times the same region with perf_counter).
* `Session` is the resident form of the same thing for callers that do not
  want the upload/download around every `run`.

Diagnostics (`macro`, `diagnostics`, `check_finite`, the per-step probe)
execute on the device too; there is no CPU compute path in this package.
"""

import contextlib
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import boundaries
from .fields import Layout, PopulationField, Precision, convert_precision
from .kernels import BACKEND, KernelPlan, pinned_empty  # noqa: F401  (BACKEND: API parity)
from .lattice import Q, RelaxationParams, equilibrium


MAGIC = b"MLB2"
VERSION = 2
# magic, version, nx, ny, nz, precision code, layout code, Q, reserved, timestep
_HEADER = struct.Struct("<4sIIIIBBBBQ")


class DivergenceError(RuntimeError):
    """Raised when a safety check finds non-finite populations."""


@dataclass
class Schedule:
    """Traversal policy: 'auto' or 'tiled' with explicit tile sizes.

    On the GPU a tile's x extent selects the thread-block width; like the
    reference's tiles it is a pure performance knob and never changes bits.
    """

    kind: str = "auto"
    tx: int = 0
    ty: int = 0
    tz: int = 1

    def __post_init__(self):
        if self.kind not in ("auto", "tiled"):
            raise ValueError(f"unknown schedule '{self.kind}'")
        if self.kind == "tiled" and (self.tx < 1 or self.ty < 1 or self.tz < 1):
            raise ValueError("tiled schedule needs positive tile sizes")

    def resolve(self, nx, ny, nz, layout):
        if self.kind == "auto":
            return None
        if self.tx > nx or self.ty > ny or self.tz > nz:
            raise ValueError(f"tile {self.tx}x{self.ty}x{self.tz} exceeds the "
                             f"{nx}x{ny}x{nz} grid")
        return (self.tx, self.ty, self.tz)

    def label(self):
        return ("auto" if self.kind == "auto"
                else f"tiled({self.tx},{self.ty},{self.tz})")


@dataclass
class RunConfig:
    """Everything a run needs beyond the initial state."""

    steps: int
    precision: Precision = Precision.SINGLE
    layout: Layout = Layout.ROW
    schedule: Schedule = field(default_factory=Schedule)
    threads: int = 0  # accepted for API parity; the GPU path has no thread pool
    output_every: int = 0
    checkpoint_every: int = 0
    out_dir: str = "out"
    device: int | None = None
    inplace: bool = False  # one device block instead of two (AA pattern)
    # z-slab decomposition over torch.distributed (one rank per GPU): None =
    # automatically when a process group with more than one rank is initialised
    distributed: bool | None = None
    gather: bool = True          # distributed runs: every rank ends with the whole host state
    transport: str = "peer"      # distributed runs: "peer" (fused peer stores) or "nccl"
    # A run on a host-resident state is upload, steps, download.  None / True: when
    # nothing has to look at the state in between (no hooks, no probe, two blocks, not
    # resident) the three phases are overlapped chunk by chunk (mlb_run_steps_host);
    # RunStats.seconds is then the device time of the WHOLE pipelined call, transfers
    # included, and RunStats.overlapped says so.  False: always upload, loop, download.
    overlap_io: bool | None = None

    def __post_init__(self):
        if self.steps < 1:
            raise ValueError("steps must be >= 1")
        for name in ("threads", "output_every", "checkpoint_every"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")


@dataclass
class SimState:
    """Populations, geometry, and physics of one simulation (host view)."""

    f_pre: PopulationField
    f_post_: PopulationField | None
    mask: np.ndarray
    nx: int
    ny: int
    nz: int
    layout: Layout
    precision: Precision
    t: int = 0
    params: RelaxationParams | None = None
    wall_u: tuple = (0.0, 0.0, 0.0)
    inlet_u: float = 0.0
    case: str = ""
    session: "Session | None" = field(default=None, repr=False)

    @property
    def f_post(self):
        """The second buffer.  Both buffers start identical (engine.py:148);
        the host copy is materialised on first use so a state that only ever
        steps on the GPU never pays for it."""
        if self.f_post_ is None:
            post = PopulationField(
                pinned_empty(self.f_pre.data.shape, self.f_pre.data.dtype),
                self.nx, self.ny, self.nz, self.layout)
            if (self.session is not None and self.session.host_stale
                    and not self.session.inplace):
                self.session.plan.download(self.session.post, post.data)
            else:
                if self.session is not None:
                    self.session.sync_host()
                np.copyto(post.data, self.f_pre.data)
            self.f_post_ = post
        return self.f_post_

    def swap(self):
        self.f_pre, self.f_post_ = self.f_post, self.f_pre
        if self.session is not None and not self.session.inplace:
            self.session.pre, self.session.post = self.session.post, self.session.pre

    def _session_for_diagnostics(self):
        if self.session is not None:
            return self.session, False
        omega = self.params.omega if self.params is not None else 1.0
        plan = KernelPlan(self.nx, self.ny, self.nz, self.layout, self.precision,
                          self.mask, omega, self.wall_u, inlet_u=self.inlet_u)
        return Session(self, plan), True

    def macro(self):
        """Density and velocity as float64 a[x, y, z] grids (engine.py:104-118),
        computed by the CUDA macro kernel."""
        sess, temp = self._session_for_diagnostics()
        try:
            sess.normalize()
            out = tuple(t.cpu().numpy().transpose(2, 1, 0)
                        for t in sess.plan.macro(sess.pre))
        finally:
            if temp:
                sess.close(sync=False)
        return out

    def diagnostics(self):
        """Total mass, momentum, kinetic energy, max |u|, non-finite count,
        fluid cells - deterministic device reductions."""
        sess, temp = self._session_for_diagnostics()
        try:
            sess.normalize()
            return sess.plan.diagnostics(sess.pre)
        finally:
            if temp:
                sess.close(sync=False)

    def fluid_cells(self):
        return int(np.count_nonzero(self.mask == boundaries.FLUID))

    def check_finite(self):
        if self.diagnostics()["nonfinite"] != 0:
            raise DivergenceError(f"divergence at step {self.t}")


def state_from_macroscopic(rho, ux, uy, uz, mask_grid, layout, precision,
                           params=None, wall_u=(0.0, 0.0, 0.0), inlet_u=0.0,
                           case=""):
    """Build a state from a[x, y, z] macroscopic grids at local equilibrium.

    Initial populations are evaluated in float64 and converted once to the
    storage precision under the strict overflow policy (engine.py:128-153).
    Scalars are accepted for uniform fields: the nineteen equilibrium
    values are then computed once and broadcast, which is the same
    arithmetic on the same inputs per cell.
    """
    mask_grid = np.asarray(mask_grid, dtype=np.uint8)
    nx, ny, nz = mask_grid.shape
    n = nx * ny * nz
    data = pinned_empty((Q, n), precision.storage)
    if all(np.ndim(a) == 0 for a in (rho, ux, uy, uz)):
        feq = equilibrium(float(rho), float(ux), float(uy), float(uz))
        stored = convert_precision(feq, precision.storage, policy="strict")
        for i in range(Q):
            data[i].fill(stored[i])
    else:
        rho, ux, uy, uz = (np.broadcast_to(np.asarray(a, dtype=np.float64),
                                           (nx, ny, nz)) for a in (rho, ux, uy, uz))
        view = data.reshape(Q, nz, ny, nx)
        for z in range(nz):  # plane by plane keeps the float64 temporaries small
            feq = equilibrium(rho[:, :, z], ux[:, :, z], uy[:, :, z], uz[:, :, z])
            stored = convert_precision(feq, precision.storage, policy="strict")
            view[:, z] = stored.transpose(0, 2, 1)
    f_pre = PopulationField(data, nx, ny, nz, layout)
    # (the flags in page-locked memory too: they are uploaded at the start of every run)
    mask = pinned_empty((nx * ny * nz,), np.uint8)
    np.copyto(mask.reshape(nz, ny, nx), mask_grid.transpose(2, 1, 0))
    return SimState(
        f_pre=f_pre, f_post_=None, mask=mask,
        nx=nx, ny=ny, nz=nz, layout=layout, precision=precision,
        params=params, wall_u=tuple(wall_u), inlet_u=float(inlet_u), case=case)


def build_plan(state, config, defer_flags=False):
    """KernelPlan for a state (engine.py:183-190), same error behaviour."""
    if state.params is None:
        raise ValueError("state has no relaxation parameters attached")
    if state.params.has_source:
        raise ValueError("the fused kernel runs the zero-source path only")
    tile = config.schedule.resolve(state.nx, state.ny, state.nz, state.layout)
    return KernelPlan(state.nx, state.ny, state.nz, state.layout, state.precision,
                      state.mask, state.params.omega, state.wall_u, tile,
                      inlet_u=state.inlet_u, device=config.device,
                      defer_flags=defer_flags)


@contextlib.contextmanager
def _hooks_read_only(state):
    """While a hook runs inside `run` the DEVICE holds the state the next step
    continues from, so an edit of the host arrays would be silently lost (the
    reference, all on the host, would step on from it).  The hook therefore
    sees READ-ONLY views: an editing hook fails loudly ("assignment
    destination is read-only") instead of being ignored;
    `state.session.host_edit()` is the way to edit a resident state."""
    fields = [f for f in (state.f_pre, state.f_post_) if f is not None]
    kept = [f.data for f in fields]
    for f in fields:
        view = f.data.view()
        view.flags.writeable = False
        f.data = view
    try:
        yield
    finally:
        for f, data in zip(fields, kept):
            f.data = data


class Session:
    """A state resident on the GPU: two device blocks and the plan.

    `attach` uploads the host arrays; stepping marks them stale; `sync_host`
    downloads.  If the host never materialised its second buffer, the device
    one is filled by a device-to-device copy (both start identical by
    construction) and is not downloaded.
    """

    def __init__(self, state, plan, inplace=False):
        self.state = state
        self.plan = plan
        self.inplace = bool(inplace)
        self.pre = plan.alloc()
        self.post = None if self.inplace else plan.alloc()
        self.host_stale = False
        self.carries_both = False
        self.upload()

    def normalize(self):
        """In-place sessions: bring the block to the normal representation
        (a no-op after an even number of steps)."""
        if self.inplace:
            self.plan.normalize(self.pre)

    def upload(self):
        st = self.state
        self.plan.upload(st.f_pre.data, self.pre)   # asynchronous (pinned host block)
        self.plan.ensure_flags()                    # flag tables, while the DMA runs
        if self.inplace:
            self.pre.repr = 0
            self.host_stale = False
            return
        if st.f_post_ is None:
            self.post.tensor.copy_(self.pre.tensor)
            same = True
        else:
            self.plan.upload(st.f_post_.data, self.post)
            nx = self.plan.nx
            same = bool(torch.equal(self.pre.tensor[:, 1:-1, :, :nx],
                                    self.post.tensor[:, 1:-1, :, :nx]))
        # Pass-through stores (full-line writes at walls) are only valid when
        # the two buffers agree on non-fluid cells; identical buffers - what
        # every state built by this package starts from (engine.py:148 of the
        # reference) - are a sufficient condition that is cheap to establish.
        # Otherwise - or when the geometry chains outlet cells, where the
        # reference's result depends on stale never-written values and the
        # library refuses the mode - the strict never-written mode is used.
        # A geometry that chains outlet cells also makes the SECOND block part of
        # the state: the chained cell reads what this block held two steps ago.
        # Such a state keeps its host copy of both blocks (sync_host materialises
        # the second one), so a run split over several sessions - engine.step in
        # a loop, checkpoint and carry on - follows the reference bit for bit.
        self.carries_both = self.plan.outlets_chained
        self.plan.set_passthrough(same and not self.carries_both)
        self.host_stale = False

    def sync_host(self):
        if not self.host_stale:
            return
        st = self.state
        self.normalize()
        if self.carries_both and not self.inplace and st.f_post_ is None:
            st.f_post                                   # downloads the second block
        self.plan.download(self.pre, st.f_pre.data, sync=False)
        if st.f_post_ is not None and not self.inplace:
            self.plan.download(self.post, st.f_post_.data, sync=False)
        torch.cuda.current_stream(self.plan.device).synchronize()
        if st.f_post_ is not None and self.inplace:
            np.copyto(st.f_post_.data, st.f_pre.data)  # there is no second device block
        self.host_stale = False

    def hooks_read_only(self):
        return _hooks_read_only(self.state)

    @contextlib.contextmanager
    def host_edit(self):
        """Edit the populations of a resident state on the host:

            with state.session.host_edit() as st:
                st.f_pre.data[q, cells] = ...

        brings the host arrays up to date, hands out the writable arrays and
        uploads them again on exit (usable inside hooks)."""
        self.sync_host()
        st = self.state
        fields = [f for f in (st.f_pre, st.f_post_) if f is not None]
        kept = [f.data for f in fields]
        for f in fields:
            base = f.data
            while not base.flags.writeable and isinstance(base.base, np.ndarray):
                base = base.base
            f.data = base
        try:
            yield st
        finally:
            self.upload()
            for f, data in zip(fields, kept):
                f.data = data

    def advance(self, nsteps, timed=False):
        """`nsteps` x (fused update, open-boundary pass, swap)."""
        if self.inplace:
            ms = self.plan.run_steps_inplace(self.pre, nsteps, timed)
        else:
            newest, other, ms = self.plan.run_steps(self.pre, self.post, nsteps, timed)
            self.pre, self.post = newest, other
        self.state.t += nsteps
        self.host_stale = True
        return ms

    def close(self, sync=True):
        if sync:
            self.sync_host()
        if self.state.session is self:
            self.state.session = None
        self.pre = self.post = None
        self.plan.close()


def open_session(state, config=None):
    """Make `state` GPU-resident (uploads it) and return the session."""
    if state.session is not None:
        return state.session
    config = config or RunConfig(steps=1, precision=state.precision,
                                 layout=state.layout)
    state.session = Session(state, build_plan(state, config, defer_flags=True),
                            inplace=config.inplace)
    return state.session


def step(state, config=None, plan=None, open_pass=None):
    """Advance the state one time step (engine.py:193-205).

    Convenience form: makes the state resident if it is not, steps once and
    brings the host arrays up to date, so callers written against the
    reference see the new populations in `state.f_pre.data`.
    """
    own = state.session is None
    sess = open_session(state, config)
    sess.advance(1)
    sess.sync_host()
    if own:
        sess.close()
    return state


@dataclass
class RunStats:
    steps: int
    seconds: float
    nx: int
    ny: int
    nz: int
    mlups: float
    probe_series: np.ndarray | None = None
    probe_samples: np.ndarray | None = None
    transport: str | None = None  # distributed runs: how the halos travelled
    overlapped: bool = False      # seconds covers upload + steps + download, pipelined


def run(state, config, on_output=None, on_checkpoint=None, probe=None):
    """Run `config.steps` steps, timing only the update loop (engine.py:208-275).

    Hooks fire on multiples of their cadence: output hooks at every multiple
    including the final step, checkpoint hooks only mid-run.  A finite check
    runs at output cadence and raises DivergenceError on NaN/inf.  When
    `probe` is an (x, y, z) cell its velocity is sampled every step on the
    device; `RunStats.probe_series` is the y-velocity series as in the
    reference, `probe_samples` the full (steps, 4) rho/u record.
    """
    if _wants_slabs(config):
        return _run_slabs(state, config, on_output, on_checkpoint, probe)
    own = state.session is None
    if (own and config.overlap_io is not False and not config.inplace and probe is None
            and not config.output_every and not config.checkpoint_every
            and state.f_post_ is None and _closed_in_z(state)):
        return _run_host_pipelined(state, config)
    if not own and state.session.inplace != bool(config.inplace):
        raise ValueError(
            f"state is resident with inplace={state.session.inplace} but the run asks for "
            f"inplace={bool(config.inplace)}: close the session first (state.session.close())")
    if not own:
        tile = config.schedule.resolve(state.nx, state.ny, state.nz, state.layout)
        if tile is not None and tuple(tile) != tuple(state.session.plan.tile):
            raise ValueError(
                f"state is resident with tile {state.session.plan.tile} but the run asks for "
                f"{tuple(tile)}: close the session first (state.session.close())")
    sess = open_session(state, config)
    if not own and not sess.host_stale:
        # A resident state whose host arrays are current: the caller may have
        # edited them, so they are the truth at the start of a run (as in the
        # reference).  When the DEVICE holds the newest populations (steps were
        # advanced since the last sync) it is the truth and nothing is uploaded.
        sess.upload()
    plan = sess.plan
    dev = plan.device
    end_t = state.t + config.steps
    samples = (torch.zeros((config.steps, 4), dtype=torch.float64, device=dev)
               if probe is not None else None)
    events = []
    done = 0
    try:
        while done < config.steps:
            chunk = config.steps - done
            if probe is not None:
                chunk = 1
            for every in (config.output_every, config.checkpoint_every):
                if every:
                    chunk = min(chunk, every - state.t % every)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(dev))
            sess.advance(chunk)
            e1.record(torch.cuda.current_stream(dev))
            events.append((e0, e1))
            done += chunk
            if samples is not None:
                sess.normalize()
                plan.probe(sess.pre, probe[0], probe[1], probe[2], samples[done - 1])
            if config.output_every and state.t % config.output_every == 0:
                state.check_finite()
                if on_output is not None:
                    sess.sync_host()
                    with sess.hooks_read_only():
                        on_output(state)
            if (config.checkpoint_every and state.t < end_t
                    and state.t % config.checkpoint_every == 0):
                if on_checkpoint is not None:
                    sess.sync_host()
                    with sess.hooks_read_only():
                        on_checkpoint(state)
        sess.sync_host()
        torch.cuda.current_stream(dev).synchronize()
    except BaseException:
        # leave the host arrays at the step `state.t` names (the reference's
        # diverged populations are visible in state.f_pre at the reported step)
        try:
            sess.sync_host()
        except Exception:
            pass
        raise
    finally:
        if own:
            sess.close(sync=False)
    seconds = sum(a.elapsed_time(b) for a, b in events) * 1e-3
    updates = state.nx * state.ny * state.nz * config.steps
    mlups = updates / (seconds * 1e6) if seconds > 0.0 else float("inf")
    rec = samples.cpu().numpy() if samples is not None else None
    return RunStats(steps=config.steps, seconds=seconds, nx=state.nx, ny=state.ny,
                    nz=state.nz, mlups=mlups,
                    probe_series=(rec[:, 2].copy() if rec is not None else None),
                    probe_samples=rec)


def _closed_in_z(state):
    """Planes 0 and nz-1 are walls and the domain is deep enough to be cut into
    at least four chunks of 1 MB or more per population: what the overlapped host
    run needs (mlb_run_steps_host; the library applies the same rule)."""
    nz, plane = state.nz, state.nx * state.ny
    if nz < 4:
        return False
    m = state.mask.reshape(nz, plane)
    walls = (boundaries.SOLID, boundaries.MOVING_WALL)
    if not (np.isin(m[0], walls).all() and np.isin(m[-1], walls).all()):
        return False
    item = state.precision.storage.itemsize
    line = 128 // item
    xp = -(-state.nx // line) * line
    cz = max(-(-nz // 128), -(-(1 << 20) // (state.ny * xp * item)))
    return -(-nz // min(cz, nz)) >= 4


def _run_host_pipelined(state, config):
    """`run` for a host-resident state that nothing looks at before the end: one
    library call uploads, steps and downloads, overlapped chunk by chunk when
    the domain is closed in z (include/mlb.h, mlb_run_steps_host); otherwise
    the same call performs the plain sequence.  Same bits either way."""
    plan = build_plan(state, config, defer_flags=True)
    try:
        a, b = plan.alloc(), plan.alloc()
        data = state.f_pre.data
        _, other, ms, overlapped = plan.run_host(data, data, a, b, config.steps)
        if plan.outlets_chained:
            # the second block is part of such a state (see Session.upload)
            plan.download(other, state.f_post.data)
        del a, b, other
    finally:
        plan.close()
    state.t += config.steps
    seconds = ms * 1e-3
    updates = state.nx * state.ny * state.nz * config.steps
    mlups = updates / (seconds * 1e6) if seconds > 0.0 else float("inf")
    return RunStats(steps=config.steps, seconds=seconds, nx=state.nx, ny=state.ny,
                    nz=state.nz, mlups=mlups, overlapped=overlapped)


def _wants_slabs(config):
    if config.distributed is False:
        return False
    import torch.distributed as dist
    on = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    if config.distributed and not on:
        raise ValueError("RunConfig(distributed=True) needs an initialised torch.distributed "
                         "process group with more than one rank (launch with torchrun)")
    return on


def _same_job_on_every_rank(state, config):
    """The slab run treats the ranks' states as ONE global domain.  A process
    group may exist for other reasons (a sweep with one simulation per rank):
    decompose only if every rank holds the same problem, else raise on all."""
    import hashlib
    import torch.distributed as dist
    p = state.params
    card = (state.nx, state.ny, state.nz, state.t, state.precision.token,
            None if p is None else float(p.omega), tuple(float(v) for v in state.wall_u),
            float(state.inlet_u), int(config.steps), bool(config.inplace),
            hashlib.blake2b(np.ascontiguousarray(state.mask), digest_size=16).hexdigest())
    cards = [None] * dist.get_world_size()
    dist.all_gather_object(cards, card)
    if any(c != cards[0] for c in cards):
        raise ValueError(
            "engine.run found a torch.distributed process group but the ranks hold different "
            "problems (shape, step, physics or mask differ), so this is not one z-decomposed "
            "domain: pass RunConfig(distributed=False) to run one simulation per rank")


def _run_slabs(state, config, on_output, on_checkpoint, probe):
    """`run` under torch.distributed: the SAME call, one rank per GPU.

    Every rank holds the (global) host state, as the reference's driver
    does; rank r uploads and advances only its z-slab [z0, z1) - 1-D slabs,
    5-population halos, the exchange fused into the boundary-plane kernel
    over peer memory (slab.PeerRing) or send/recv - and the loop body,
    hook cadence, finite check and timing are those of the single-GPU run.
    Before a hook fires, and at the end, each rank downloads its slab into
    its part of the host arrays; with `config.gather` the slabs are then
    broadcast so that every rank sees the whole state (switch it off for
    domains whose host copy is only ever looked at slab-wise).
    RunStats.seconds is the device time of the loop, max over ranks.
    """
    import torch.distributed as dist
    from . import slab
    if state.session is not None:
        state.session.close()
    if state.params is None:
        raise ValueError("state has no relaxation parameters attached")
    if state.params.has_source:
        raise ValueError("the fused kernel runs the zero-source path only")
    rank, world = dist.get_rank(), dist.get_world_size()
    _same_job_on_every_rank(state, config)
    nx, ny, nz = state.nx, state.ny, state.nz
    z0, z1 = slab.partition(nz, world)[rank]
    n = z1 - z0
    flags = state.mask.reshape(nz, ny, nx)
    lo, hi = slab.slab_halo_flags(flags, nx, ny, z0, z1)
    tile = config.schedule.resolve(nx, ny, n, state.layout)
    # (a slab the library refuses - e.g. an outlet cell at x = 0 in this rank's planes only -
    # must stop EVERY rank, not leave the others waiting in the next collective)
    plan, refused = None, None
    try:
        plan = KernelPlan(nx, ny, n, state.layout, state.precision, flags[z0:z1], state.params.omega,
                          state.wall_u, tile, inlet_u=state.inlet_u, device=config.device,
                          halo_lo=lo, halo_hi=hi, slab=True)
    except (ValueError, MemoryError) as exc:
        refused = exc
    here = torch.device("cuda", torch.cuda.current_device() if config.device is None
                        else int(config.device))
    if not slab._agree(refused is None, world, None, here):
        if plan is not None:
            plan.close()
        raise ValueError("engine.run: the slab of some rank was refused"
                         + (f" (this rank: {refused})" if refused else ""))
    dev = plan.device
    dense = state.f_pre.data.reshape(Q, nz, ny, nx)
    mine = pinned_empty((Q, n * ny * nx), state.precision.storage)   # this rank's slab, contiguous
    np.copyto(mine.reshape(Q, n, ny, nx), dense[:, z0:z1])
    a = plan.alloc()
    plan.upload(mine, a)
    mine2, carry = None, False
    if config.inplace:
        # one block per rank (AA pattern over peer memory)
        b = None
        runner, transport = slab.open_inplace_runner(plan, a, rank, world), "peer"
    else:
        b = plan.alloc()
        same = state.f_post_ is None
        if same:
            b.tensor.copy_(a.tensor)        # both blocks identical (engine.py:148)
        else:
            # the host holds a second buffer: it is part of the state (engine.py:89)
            mine2 = pinned_empty((Q, n * ny * nx), state.precision.storage)
            np.copyto(mine2.reshape(Q, n, ny, nx),
                      state.f_post_.data.reshape(Q, nz, ny, nx)[:, z0:z1])
            plan.upload(mine2, b)
            same = bool(torch.equal(a.tensor[:, 1:-1, :, :nx], b.tensor[:, 1:-1, :, :nx]))
        chained = plan.outlets_chained
        plan.set_passthrough(same and not chained)      # per slab: never changes bits
        # Chained outlet cells read stale values of the second block (Session.upload), and a
        # second buffer that differs from the first is state too: if ANY rank has either, every
        # rank brings its second block back to the host arrays as well (collective decision).
        carry = not slab._agree(same and not chained, world, None, here)
        runner, transport = slab.open_runner(plan, a, b, rank, world, transport=config.transport)
    pre, post = a, b

    fence = False

    def advance(k):
        nonlocal pre, post, fence
        if config.inplace:
            # In place the neighbours' next pull half writes into THIS rank's
            # boundary planes (not into halo planes nobody else reads): whatever
            # read the block since the last settle() - probe, diagnostics,
            # download - must be over on every rank before anyone steps on.
            if fence:
                runner.fence()
                fence = False
            runner.run_inplace(pre, k)
        else:
            pre, post = runner.run(pre, post, k)

    def settle():
        """Before anything reads the block: pushes landed, normal representation."""
        nonlocal fence
        if config.inplace:
            runner.normalize(pre)
            fence = True
        else:
            runner.finish()

    def sync_host():
        """This rank's slab into the host arrays; all slabs with config.gather."""
        nonlocal mine2
        blocks = [(pre, mine, dense)]
        if carry:
            if mine2 is None:
                mine2 = pinned_empty((Q, n * ny * nx), state.precision.storage)
            blocks.append((post, mine2, state.f_post.data.reshape(Q, nz, ny, nx)))
        parts = slab.partition(nz, world)
        biggest = max(e - s for s, e in parts)
        for blk, stage, whole in blocks:
            plan.download(blk, stage)
            np.copyto(whole[:, z0:z1], stage.reshape(Q, n, ny, nx))
            if not config.gather:
                continue
            scratch = torch.empty((Q, biggest, ny, nx), dtype=blk.tensor.dtype, device=dev)
            own = blk.tensor[:, 1:-1, :, :nx].contiguous()
            for r, (s0, s1) in enumerate(parts):
                buf = own if r == rank else scratch[:, :s1 - s0].contiguous()
                dist.broadcast(buf, src=r)
                if r != rank:
                    np.copyto(whole[:, s0:s1], buf.cpu().numpy())
        if state.f_post_ is not None and not carry:
            np.copyto(state.f_post_.data, state.f_pre.data)

    owner = probe is not None and z0 <= probe[2] < z1
    samples = (torch.zeros((config.steps, 4), dtype=torch.float64, device=dev)
               if probe is not None else None)
    end_t = state.t + config.steps
    events, done = [], 0
    try:
        while done < config.steps:
            chunk = config.steps - done
            if probe is not None:
                chunk = 1
            for every in (config.output_every, config.checkpoint_every):
                if every:
                    chunk = min(chunk, every - state.t % every)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(dev))
            advance(chunk)
            e1.record(torch.cuda.current_stream(dev))
            events.append((e0, e1))
            state.t += chunk
            done += chunk
            if probe is not None and config.inplace:
                settle()            # collective: every rank, not only the probe's owner
            if owner:
                plan.probe(pre, probe[0], probe[1], probe[2] - z0, samples[done - 1])
            hook_out = config.output_every and state.t % config.output_every == 0
            hook_ckp = (config.checkpoint_every and state.t < end_t
                        and state.t % config.checkpoint_every == 0)
            if hook_out or hook_ckp:
                settle()
            if hook_out:
                total = slab.combine_diagnostics(plan.diagnostics(pre), rank, world)
                if total["nonfinite"] != 0:
                    raise DivergenceError(f"divergence at step {state.t}")
                if on_output is not None:
                    sync_host()
                    with _hooks_read_only(state):
                        on_output(state)
            if hook_ckp and on_checkpoint is not None:
                sync_host()
                with _hooks_read_only(state):
                    on_checkpoint(state)
        settle()
        sync_host()
        torch.cuda.synchronize(dev)
        ms = torch.tensor([sum(x.elapsed_time(y) for x, y in events)], dtype=torch.float64,
                          device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        rec = None
        if samples is not None:
            # the rank that owns the probe cell holds the series; everyone gets it
            src = next(r for r, (s, e) in enumerate(slab.partition(nz, world)) if s <= probe[2] < e)
            dist.broadcast(samples, src=src)
            rec = samples.cpu().numpy()
    finally:
        if runner.ring is not None:
            runner.ring.close()
        plan.close()
    seconds = float(ms.item()) * 1e-3
    updates = nx * ny * nz * config.steps
    mlups = updates / (seconds * 1e6) if seconds > 0.0 else float("inf")
    return RunStats(steps=config.steps, seconds=seconds, nx=nx, ny=ny, nz=nz, mlups=mlups,
                    probe_series=(rec[:, 2].copy() if rec is not None else None),
                    probe_samples=rec, transport=transport)


def checkpoint(state, path):
    """Write the state in the binary checkpoint format, version 2.

    The reference's MLB1 format (engine.py:9-13, :278-287) with the third
    dimension added: little-endian header `<4sIIIIBBBBQ` = magic "MLB2", u32
    version 2, u32 nx, ny, nz, u8 precision code, u8 layout code, u8 Q (19),
    u8 reserved, u64 timestep (32 bytes), then the nineteen pre-buffer planes
    in cell order, then the mask, one byte per cell.  Physics parameters
    are not serialised.  A GPU-resident state is synchronised first.
    """
    if state.session is not None:
        state.session.sync_host()
    le_storage = state.precision.storage.newbyteorder("<")
    planes = np.ascontiguousarray(state.f_pre.data, dtype=le_storage)
    header = _HEADER.pack(MAGIC, VERSION, state.nx, state.ny, state.nz,
                          state.precision.code, state.layout.code, Q, 0, state.t)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(planes.tobytes())
        fh.write(np.ascontiguousarray(state.mask, dtype=np.uint8).tobytes())


def restore(path):
    """Read a checkpoint back into a host state (engine.py:290-330).

    The returned state carries params=None; callers re-attach physics with
    `cases.attach_params`.  Header and payload sizes are validated and
    errors name the offending byte offset.
    """
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HEADER.size:
        raise ValueError(
            f"truncated checkpoint: {len(blob)} bytes is shorter than the "
            f"{_HEADER.size}-byte header")
    magic, version, nx, ny, nz, pcode, lcode, q, _, t = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise ValueError(f"not a checkpoint file (magic {magic!r} at offset 0)")
    if version != VERSION:
        raise ValueError(f"unsupported checkpoint version {version} "
                         f"(offset 4), expected {VERSION}")
    precision = Precision.from_code(pcode)
    layout = Layout.from_code(lcode)
    if q != Q:
        raise ValueError(f"checkpoint holds {q} populations per cell "
                         f"(offset 22), expected {Q}")
    n = nx * ny * nz
    le_storage = precision.storage.newbyteorder("<")
    plane_bytes = Q * n * le_storage.itemsize
    expected = _HEADER.size + plane_bytes + n
    if len(blob) != expected:
        raise ValueError(
            f"checkpoint payload mismatch for declared {nx}x{ny}x{nz} grid: "
            f"expected {expected} bytes, found {len(blob)} "
            f"(payload starts at offset {_HEADER.size})")
    planes = np.frombuffer(blob, dtype=le_storage, count=Q * n, offset=_HEADER.size)
    data = pinned_empty((Q, n), precision.storage)
    data[:] = planes.reshape(Q, n)
    mask = np.frombuffer(blob, dtype=np.uint8, count=n,
                         offset=_HEADER.size + plane_bytes).copy()
    if mask.max(initial=0) > boundaries.OUTLET:
        raise ValueError("checkpoint mask holds unknown cell codes")
    f_pre = PopulationField(data, nx, ny, nz, layout)
    return SimState(f_pre=f_pre, f_post_=None, mask=mask, nx=nx, ny=ny, nz=nz,
                    layout=layout, precision=precision, t=t)
