"""The plugin boundary: `KernelPlan.step(fpre, fpost)` on CUDA.

Host-side mirror of /root/reference/pkg/src/lb2d/kernels.py:398-462.  The
reference's KernelPlan captures shape, precision, tile, wall velocity and
relaxation rate and owns the backend machinery; `.step(fpre, fpost)` reads
`fpre` and writes every fluid cell of `fpost` exactly once.  This one has
the same shape (plus `nz`, a 3-component wall velocity, the inlet velocity
the open-boundary pass needs, and a device), but its backend machinery is an
opaque `mlb_plan*` from libmlb_d3q19.so (include/mlb.h) launching
hand-written sm_100a kernels.  PyTorch appears here only as the owner of
device buffers and streams: raw `data_ptr()` / `cuda_stream` values are all
that cross the C ABI.

`.step` accepts either the reference's HOST blocks - C-contiguous
`(19, nx*ny*nz)` numpy arrays of the storage dtype, x fastest - in which
case it is a synchronous upload / step / download like the reference call,
or `DeviceField`s (the padded device layout), in which case it enqueues on
the current CUDA stream and returns.

Backend selection mirrors kernels.py:41-55: the environment variable
`MLB_BACKEND` may be 'auto' or 'cuda'; anything else is a ValueError.
There is exactly one backend and no CPU fallback.
"""

import ctypes
import os

import numpy as np
import torch

from . import _cabi
from .fields import Layout, Precision
from .lattice import Q


def _pick_backend():
    token = os.environ.get("MLB_BACKEND", "auto").strip().lower() or "auto"
    if token in ("auto", "cuda"):
        return "cuda"
    raise ValueError(f"MLB_BACKEND must be 'auto' or 'cuda', got '{token}'")


BACKEND = _pick_backend()

_BLOCK_WIDTHS = (32, 64, 128, 256, 512)


def _stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _host_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class _LibBlock:
    """`nbytes` of cudaMalloc memory from the library (mlb_block_alloc), seen by
    torch through `__cuda_array_interface__`.  The z-slab exchange exports
    population blocks over CUDA IPC, which needs plain cudaMalloc allocations:
    taking them from the library keeps that independent of how torch's caching
    allocator is configured (expandable segments, cudaMallocAsync).  The tensor
    made from this object keeps it alive; the memory goes back to the library
    when the last reference dies."""

    def __init__(self, lib, device_index, nbytes, shape, typestr):
        ptr = ctypes.c_void_p()
        _cabi.check(lib.mlb_block_alloc(int(device_index), int(nbytes), ctypes.byref(ptr)))
        self._lib, self.ptr, self.nbytes = lib, ptr.value, int(nbytes)
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (self.ptr, False), "strides": None,
                                         "version": 2}

    def __del__(self):
        ptr, self.ptr = getattr(self, "ptr", None), None
        if ptr:
            try:
                self._lib.mlb_block_free(ctypes.c_void_p(ptr))
            except Exception:   # interpreter shutdown
                pass


class DeviceField:
    """One population block in the padded device layout; torch views memory
    the library allocated (`KernelPlan.alloc`).

    `tensor` has shape (19, nz+2, ny, xp); storage plane 0 and nz+1 are the
    halo planes, slab plane lz is storage plane lz+1, xp is nx rounded up
    to a whole number of 128-byte lines (include/mlb.h).
    """

    def __init__(self, tensor, nx, ny, nz):
        self.tensor = tensor
        self.nx, self.ny, self.nz = nx, ny, nz
        self.repr = 0  # in-place runs only: 0 = normal, 1 = shifted (include/mlb.h)

    @property
    def ptr(self):
        return ctypes.c_void_p(self.tensor.data_ptr())

    def plane(self, q, lz):
        """View of population q, slab plane lz (-1 and nz are the halos)."""
        return self.tensor[q, lz + 1]


class KernelPlan:
    """Everything one run needs to advance the populations one step."""

    def __init__(self, nx, ny, nz, layout, precision, mask, omega,
                 wall_u=(0.0, 0.0, 0.0), tile=None, backend=None, *,
                 inlet_u=0.0, device=None, halo_lo=None, halo_hi=None,
                 slab=False, defer_flags=False):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        if layout is not Layout.ROW:
            raise ValueError("the CUDA path stores x fastest (Layout.ROW) only")
        self.layout = layout
        if not isinstance(precision, Precision):
            precision = Precision.from_token(precision)
        self.precision = precision
        self.backend = backend or BACKEND
        if self.backend != "cuda":
            raise ValueError(f"unknown backend '{self.backend}'")
        self.sx, self.sy, self.sz = layout.strides(self.nx, self.ny, self.nz)
        auto_tile = tile is None
        if auto_tile:
            tile = (min(self.nx, 128), 1, 1)  # one contiguous line segment per block
        tile = tuple(int(t) for t in tile) + (1,) * (3 - len(tile))
        tx, ty, tz = tile
        if not (1 <= tx <= self.nx and 1 <= ty <= self.ny and 1 <= tz <= self.nz):
            raise ValueError(f"tile {tx}x{ty}x{tz} does not fit a "
                             f"{self.nx}x{self.ny}x{self.nz} grid")
        self.tile = tile
        mask = np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        if mask.size != self.nx * self.ny * self.nz:
            raise ValueError(f"mask has {mask.size} cells, expected "
                             f"{self.nx * self.ny * self.nz}")
        self.mask = mask
        self.wall_u = tuple(float(v) for v in wall_u) + (0.0,) * (3 - len(wall_u))
        self.inlet_u = float(inlet_u)
        self.omega = float(omega)
        self.slab = bool(slab)

        lib = _cabi.lib()  # raises RuntimeError if the extension is not built
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device is visible; the D3Q19 path has "
                               "no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else int(device))
        self._lib = lib
        self._plan = ctypes.c_void_p()
        uw = (ctypes.c_double * 3)(*self.wall_u)
        _cabi.check(lib.mlb_plan_create(
            ctypes.byref(self._plan), self.nx, self.ny, self.nz, precision.code,
            self.omega, uw, self.inlet_u, self.device.index,
            _cabi.MLB_Z_HALO if self.slab else _cabi.MLB_Z_PERIODIC))
        self._layout = _cabi.Layout()
        _cabi.check(lib.mlb_plan_get_layout(self._plan, ctypes.byref(self._layout)))
        # schedule 'auto' lets the library pick (the vectorised kernel when
        # the row length allows, see mlb_plan_set_variant); an explicit tile
        # selects the one-cell-per-thread kernel with the largest supported
        # block width not above the tile's x extent.  Never changes bits.
        if not auto_tile:
            width = max([w for w in _BLOCK_WIDTHS if w <= max(tx, 32)])
            _cabi.check(lib.mlb_plan_set_variant(self._plan, width))

        def plane(h):
            if h is None:
                return None
            h = np.ascontiguousarray(h, dtype=np.uint8).reshape(-1)
            if h.size != self.nx * self.ny:
                raise ValueError("halo flag plane must have nx*ny cells")
            return h
        self._halo = (plane(halo_lo), plane(halo_hi))
        self._flags_set = False
        self._scratch = None
        self.passthrough = False
        # defer_flags: the caller starts its (asynchronous) population upload
        # first and calls ensure_flags() while the DMA runs
        if not defer_flags:
            self.ensure_flags()

    def ensure_flags(self):
        """Hand the flag array to the library (builds the per-cell tables on
        the device).  Idempotent."""
        if self._flags_set:
            return
        lo, hi = self._halo
        _cabi.check(self._lib.mlb_plan_set_flags(
            self._plan, _host_ptr(self.mask),
            _host_ptr(lo) if lo is not None else ctypes.c_void_p(None),
            _host_ptr(hi) if hi is not None else ctypes.c_void_p(None)))
        self._flags_set = True

    # -- lifetime ----------------------------------------------------------
    def close(self):
        plan, self._plan = getattr(self, "_plan", None), None
        if plan:
            self._lib.mlb_plan_destroy(plan)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- geometry ----------------------------------------------------------
    @property
    def xp(self):
        return int(self._layout.xp)

    @property
    def field_shape(self):
        return (Q, self.nz + 2, self.ny, self.xp)

    @property
    def field_bytes(self):
        return int(self._layout.bytes)

    def alloc(self, zero=False):
        """A caller-owned device population block: cudaMalloc memory from the
        library (exportable over CUDA IPC whatever torch's allocator is set to),
        wrapped as a torch tensor that keeps it alive."""
        typestr = {Precision.SINGLE: "<f4", Precision.DOUBLE: "<f8", Precision.MIXED1: "<f2",
                   Precision.MIXED2: "<f4"}[self.precision]
        try:
            block = _LibBlock(self._lib, self.device.index, self.field_bytes, self.field_shape,
                              typestr)
        except MemoryError:
            torch.cuda.empty_cache()   # let torch's cache go, then once more
            block = _LibBlock(self._lib, self.device.index, self.field_bytes, self.field_shape,
                              typestr)
        t = torch.as_tensor(block, device=self.device)
        if zero:
            t.zero_()
        return DeviceField(t, self.nx, self.ny, self.nz)

    def device_flags(self):
        """The flag bytes the kernel tests, read back dense, for bit-exact
        geometry checks."""
        out = np.empty(self.nx * self.ny * self.nz, dtype=np.uint8)
        _cabi.check(self._lib.mlb_plan_get_flags(self._plan, _host_ptr(out)))
        return out

    def geometry_stats(self):
        """(distinct wall-link patterns in the plan's dictionary, cells that
        overflowed it and read full-width class words)."""
        out = (ctypes.c_int64 * 2)()
        _cabi.check(self._lib.mlb_plan_geometry_stats(self._plan, out))
        return int(out[0]), int(out[1])

    def set_physics(self, omega=None, wall_u=None, inlet_u=None):
        if omega is not None:
            self.omega = float(omega)
        if wall_u is not None:
            self.wall_u = tuple(float(v) for v in wall_u) + (0.0,) * (3 - len(wall_u))
        if inlet_u is not None:
            self.inlet_u = float(inlet_u)
        uw = (ctypes.c_double * 3)(*self.wall_u)
        _cabi.check(self._lib.mlb_plan_set_physics(self._plan, self.omega, uw,
                                                   self.inlet_u))

    def set_variant(self, variant):
        """Kernel variant (tuning knob, never changes bits): 0 = auto,
        32..512 = one cell per thread with that block width, W*1000 + LX =
        packs of cells (W = 1: 16-byte packs for fp32/fp64, W = 2 / 3: 8- /
        4-byte packs for fp16 storage) with LX = 8 / 16 / 32 packs per warp
        row (include/mlb.h)."""
        _cabi.check(self._lib.mlb_plan_set_variant(self._plan, int(variant)))

    set_block_width = set_variant

    @property
    def kernel_name(self):
        return self._lib.mlb_plan_kernel_name(self._plan).decode()

    def set_passthrough(self, on):
        """Pass-through stores: also rewrite non-fluid cells of fpost with the
        value they hold in fpre.  Only valid when the two blocks agree on
        non-fluid cells (see include/mlb.h); memory then ends up identical
        to the strict never-written mode, but every store is a full line."""
        self.passthrough = bool(on)
        _cabi.check(self._lib.mlb_plan_set_passthrough(self._plan, int(self.passthrough)))

    @property
    def outlets_chained(self):
        """True when an outlet cell copies from another outlet cell: the
        reference then reads that cell's stale value in fpost (engine.py:179-180),
        so the result depends on the history of BOTH blocks.  The library
        refuses pass-through stores for exactly these geometries; that refusal
        is the query."""
        self.ensure_flags()
        was = self.passthrough
        try:
            self.set_passthrough(True)
        except ValueError:
            self.passthrough = False
            return True
        self.set_passthrough(was)
        return False

    def set_inplace_layout(self, mode):
        """Thread layout of the in-place pull half (include/mlb.h): 0 classic,
        1 row blocks, -1 auto.  Never changes bits."""
        _cabi.check(self._lib.mlb_plan_set_inplace_layout(self._plan, int(mode)))

    def set_graph(self, mode):
        """CUDA graphs in `run_steps` / `run_steps_inplace`: -1 auto (small,
        launch-bound domains), 0 never, 1 always.  Never changes bits."""
        _cabi.check(self._lib.mlb_plan_set_graph(self._plan, int(mode)))

    def set_prefetch(self, cells):
        """L2 prefetch distance of the pack kernels in cells (-1 auto, 0 off);
        a performance knob only - results never depend on it (include/mlb.h)."""
        _cabi.check(self._lib.mlb_plan_set_prefetch(self._plan, int(cells)))

    # -- host <-> device ---------------------------------------------------
    def _check_host(self, a):
        n = self.nx * self.ny * self.nz
        if not (isinstance(a, np.ndarray) and a.shape == (Q, n)
                and a.dtype == self.precision.storage and a.flags.c_contiguous):
            raise ValueError(
                f"host population block must be a C-contiguous ({Q}, {n}) "
                f"{self.precision.storage} array")

    def upload(self, host, dev):
        self._check_host(host)
        _cabi.check(self._lib.mlb_upload(self._plan, _host_ptr(host), dev.ptr,
                                         _stream_ptr(self.device)))

    def download(self, dev, host, sync=True):
        self._check_host(host)
        _cabi.check(self._lib.mlb_download(self._plan, dev.ptr, _host_ptr(host),
                                           _stream_ptr(self.device)))
        if sync:
            torch.cuda.current_stream(self.device).synchronize()

    # -- the hot path ------------------------------------------------------
    def step(self, fpre, fpost):
        """Advance one step: read fpre, write every fluid cell of fpost."""
        if isinstance(fpre, DeviceField):
            _cabi.check(self._lib.mlb_step(self._plan, fpre.ptr, fpost.ptr,
                                           _stream_ptr(self.device)))
            return
        self._check_host(fpre)
        self._check_host(fpost)
        if self._scratch is None:
            self._scratch = (self.alloc(), self.alloc())
        a, b = self._scratch
        _cabi.check(self._lib.mlb_step_host(self._plan, _host_ptr(fpre),
                                            _host_ptr(fpost), a.ptr, b.ptr,
                                            _stream_ptr(self.device)))

    def step_range(self, fpre, fpost, z0, z1):
        _cabi.check(self._lib.mlb_step_range(self._plan, fpre.ptr, fpost.ptr,
                                             int(z0), int(z1),
                                             _stream_ptr(self.device)))

    def step_open_range(self, fpre, fpost, z0, z1):
        """One time step's work on planes [z0, z1): fused update + open-
        boundary pass (fused into one kernel when possible, include/mlb.h)."""
        _cabi.check(self._lib.mlb_step_open_range(self._plan, fpre.ptr, fpost.ptr,
                                                  int(z0), int(z1),
                                                  _stream_ptr(self.device)))

    def open_pass(self, fpost):
        _cabi.check(self._lib.mlb_open_pass(self._plan, fpost.ptr,
                                            _stream_ptr(self.device)))

    def open_pass_range(self, fpost, z0, z1):
        _cabi.check(self._lib.mlb_open_pass_range(self._plan, fpost.ptr, int(z0),
                                                  int(z1), _stream_ptr(self.device)))

    def run_steps(self, a, b, nsteps, timed=False):
        """`nsteps` x (fused update, open-boundary pass, swap) on the device.

        Returns (newest, other, ms): the block holding the newest
        populations, the other one, and - when `timed` - the device time of
        the loop in milliseconds from CUDA events on the launching stream
        (the call then synchronises)."""
        ms = ctypes.c_float(0.0)
        _cabi.check(self._lib.mlb_run_steps(
            self._plan, a.ptr, b.ptr, int(nsteps), _stream_ptr(self.device),
            ctypes.byref(ms) if timed else None))
        newest, other = (a, b) if nsteps % 2 == 0 else (b, a)
        return newest, other, (ms.value if timed else None)

    def run_host(self, host_in, host_out, a, b, nsteps, chunk_planes=0):
        """A whole run on HOST blocks in one call (mlb_run_steps_host): upload
        `host_in` into `a`, `nsteps` steps over (a, b), download the newest
        populations into `host_out` (may be `host_in`) - with the three phases
        overlapped chunk by chunk when the domain is closed in z.  Hands the
        flags over on the way if `ensure_flags` has not run yet.  Synchronous.
        Returns (newest, other, ms of the whole call, overlapped?)."""
        self._check_host(host_in)
        self._check_host(host_out)
        ms, ov = ctypes.c_float(0.0), ctypes.c_int(0)
        flags = None if self._flags_set else _host_ptr(self.mask)
        if not self._flags_set and any(h is not None for h in self._halo):
            raise ValueError("run_host is for whole-domain plans (no halo flag planes)")
        _cabi.check(self._lib.mlb_run_steps_host(
            self._plan, _host_ptr(host_in), _host_ptr(host_out), a.ptr, b.ptr, int(nsteps),
            int(chunk_planes), flags, _stream_ptr(self.device), ctypes.byref(ms), ctypes.byref(ov)))
        self._flags_set = True
        newest, other = (a, b) if nsteps % 2 == 0 else (b, a)
        return newest, other, ms.value, bool(ov.value)

    def run_steps_inplace(self, f, nsteps, timed=False):
        """`nsteps` steps on ONE block (the AA pattern): same arithmetic and
        traffic as `run_steps`, half the memory.  Walls only.  `f.repr`
        tracks the representation the block is left in; call `normalize`
        before reading it back.  Returns the loop's device time in ms when
        `timed`."""
        ms = ctypes.c_float(0.0)
        r = ctypes.c_int(f.repr)
        _cabi.check(self._lib.mlb_run_steps_inplace(
            self._plan, f.ptr, int(nsteps), ctypes.byref(r), _stream_ptr(self.device),
            ctypes.byref(ms) if timed else None))
        f.repr = r.value
        return ms.value if timed else None

    def normalize(self, f):
        """Bring an in-place block back to the normal representation."""
        r = ctypes.c_int(f.repr)
        _cabi.check(self._lib.mlb_inplace_normalize(self._plan, f.ptr, ctypes.byref(r),
                                                    _stream_ptr(self.device)))
        f.repr = r.value

    def step_inplace_range(self, f, z0, z1, below, above):
        """One in-place half-step (pull if f.repr == 0, local if 1) on planes
        [z0, z1) of a z-slab; `below` / `above` = (device pointer, nz) of the
        ring neighbours' blocks.  Does not flip f.repr (the caller does, once
        all planes are done)."""
        _cabi.check(self._lib.mlb_step_inplace_range(
            self._plan, f.ptr, int(f.repr), int(z0), int(z1),
            ctypes.c_void_p(below[0]), int(below[1]), ctypes.c_void_p(above[0]), int(above[1]),
            _stream_ptr(self.device)))

    def inplace_swap_slab(self, f, above):
        """Shifted -> normal representation of a slab without a step (the halo
        planes must be refilled afterwards)."""
        _cabi.check(self._lib.mlb_inplace_swap_slab(
            self._plan, f.ptr, ctypes.c_void_p(above[0]), int(above[1]),
            _stream_ptr(self.device)))

    def halo_copy(self, dst, src, face):
        """Fill one halo plane of `dst` from the matching boundary plane of
        `src` (5 crossing populations), on this device or a peer."""
        _cabi.check(self._lib.mlb_halo_copy(self._plan, dst.ptr, src.ptr,
                                            int(src.nz), int(face),
                                            _stream_ptr(self.device)))

    def halo_push(self, src, dst_ptr, dst_nz, face):
        """The same exchange from the sender's side: the boundary plane of the
        local block `src` into the halo plane of a neighbour's block given as
        a raw device pointer (peer memory, see slab.PeerRing)."""
        _cabi.check(self._lib.mlb_halo_push(self._plan, src.ptr, ctypes.c_void_p(dst_ptr),
                                            int(dst_nz), int(face),
                                            _stream_ptr(self.device)))

    def step_push_range(self, fpre, fpost, z0, z1, below=None, above=None):
        """`step_open_range` whose boundary planes also store their crossing
        populations into the ring neighbours' halo planes from inside the
        fused kernel.  `below` / `above` are (device pointer, nz) of the
        neighbours' post blocks, or None."""
        bp, bn = below if below is not None else (None, 0)
        ap, an = above if above is not None else (None, 0)
        _cabi.check(self._lib.mlb_step_push_range(
            self._plan, fpre.ptr, fpost.ptr, int(z0), int(z1),
            ctypes.c_void_p(bp), int(bn), ctypes.c_void_p(ap), int(an),
            _stream_ptr(self.device)))

    # -- diagnostics -------------------------------------------------------
    def macro(self, dev):
        """rho, ux, uy, uz as float64 CUDA tensors of shape (nz, ny, nx)."""
        out = [torch.empty((self.nz, self.ny, self.nx), dtype=torch.float64,
                           device=self.device) for _ in range(4)]
        _cabi.check(self._lib.mlb_macro(
            self._plan, dev.ptr, *[ctypes.c_void_p(o.data_ptr()) for o in out],
            _stream_ptr(self.device)))
        return tuple(out)

    def diagnostics(self, dev):
        out = (ctypes.c_double * 8)()
        _cabi.check(self._lib.mlb_diagnostics(self._plan, dev.ptr, out,
                                              _stream_ptr(self.device)))
        keys = ("mass", "px", "py", "pz", "kinetic_energy", "max_u",
                "nonfinite", "fluid_cells")
        return dict(zip(keys, list(out)))

    def probe(self, dev, x, y, z, out4):
        """Enqueue a (rho, ux, uy, uz) sample of one cell into a 4-double
        CUDA tensor (no host round trip)."""
        _cabi.check(self._lib.mlb_probe(self._plan, dev.ptr, int(x), int(y), int(z),
                                        ctypes.c_void_p(out4.data_ptr()),
                                        _stream_ptr(self.device)))


def _torch_dtype(precision):
    return {Precision.SINGLE: torch.float32, Precision.DOUBLE: torch.float64,
            Precision.MIXED1: torch.float16, Precision.MIXED2: torch.float32}[precision]


def pinned_empty(shape, dtype):
    """A numpy array backed by page-locked host memory when CUDA is present
    (so uploads/downloads are real asynchronous DMA), plain otherwise."""
    dtype = np.dtype(dtype)
    if torch.cuda.is_available():
        tdt = {np.dtype(np.float32): torch.float32,
               np.dtype(np.float64): torch.float64,
               np.dtype(np.float16): torch.float16,
               np.dtype(np.uint8): torch.uint8}[dtype]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)
