"""TEST INFRASTRUCTURE - ctypes front end of the C oracle (d3q19_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module; the product package never
does (tests/test_no_oracle_in_product.py enforces it).

`CpuOracle` steps dense host blocks `(19, nz*ny*nx)` exactly the way the
reference's `KernelPlan.step` + `_OpenBoundaryPass.apply` step 2-D ones
(lb2d kernels.py:445-462, engine.py:176-180); `SlabOracle` does the same on
a slab block with one halo plane either side, which is what the z-slab
decomposition tests drive on CPU.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle_d3q19.so")
_SRCS = [os.path.join(_HERE, n) for n in ("d3q19_oracle.c", "d3q19_body.inc")]


class Geom(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("rs", ctypes.c_long), ("ps", ctypes.c_long), ("qs", ctypes.c_long),
                ("zoff", ctypes.c_int),
                ("zlo_src", ctypes.c_int), ("zhi_src", ctypes.c_int)]


def build(force=False):
    """Compile the oracle with the committed Makefile if missing or stale."""
    stale = (not os.path.exists(_LIB)
             or any(os.path.getmtime(s) > os.path.getmtime(_LIB) for s in _SRCS))
    if force or stale:
        subprocess.run(["make", "-C", _HERE, "-B", "liboracle_d3q19.so"],
                       check=True, capture_output=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        for suf in ("f32", "f64", "h32", "f32c64"):
            fn = getattr(_lib, f"orc_step_{suf}")
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(Geom), ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_double,
                           ctypes.POINTER(ctypes.c_double),
                           ctypes.c_int, ctypes.c_int, ctypes.c_int]
            fn = getattr(_lib, f"orc_open_pass_{suf}")
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(Geom), ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_double, ctypes.c_int, ctypes.c_int]
            fn = getattr(_lib, f"orc_macro_{suf}")
            fn.restype = None
            fn.argtypes = [ctypes.POINTER(Geom)] + [ctypes.c_void_p] * 5
            fn = getattr(_lib, f"orc_diag_{suf}")
            fn.restype = None
            fn.argtypes = [ctypes.POINTER(Geom)] + [ctypes.c_void_p] * 3
            fn = getattr(_lib, f"orc_equilibrium_{suf}")
            fn.restype = None
            fn.argtypes = [ctypes.c_double] * 4 + [ctypes.c_void_p]
    return _lib


def _suffix(dtype, compute=None):
    dtype = np.dtype(dtype)
    if dtype == np.float32 and compute is not None and np.dtype(compute) == np.float64:
        return "f32c64"  # single storage, double compute (the reference's MIXED2)
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    if dtype == np.float16:
        return "h32"  # half storage, single compute (the reference's MIXED1)
    raise ValueError(f"oracle handles float16/float32/float64 storage, got {dtype}")


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Base:
    def __init__(self, geom, flags, omega, wall_u, inlet_u, threads, compute=None):
        self.compute = compute  # None: the storage dtype's own (float16 -> float32)
        self.geom = geom
        self.flags = flags
        self.omega = float(omega)
        self._uw = (ctypes.c_double * 3)(*[float(v) for v in wall_u])
        self.inlet_u = float(inlet_u)
        self.threads = int(threads)

    def _check(self, *arrs):
        for a in arrs:
            if not (a.flags.c_contiguous and a.size == 19 * self.geom.qs):
                raise ValueError("population block has the wrong shape/strides")

    def step_range(self, fpre, fpost, z0, z1):
        self._check(fpre, fpost)
        fn = getattr(lib(), f"orc_step_{_suffix(fpre.dtype, self.compute)}")
        rc = fn(ctypes.byref(self.geom), _ptr(fpre), _ptr(fpost), _ptr(self.flags),
                self.omega, self._uw, z0, z1, self.threads)
        if rc:
            raise RuntimeError(f"orc_step failed ({rc})")

    def open_pass_range(self, fpost, z0, z1):
        self._check(fpost)
        fn = getattr(lib(), f"orc_open_pass_{_suffix(fpost.dtype, self.compute)}")
        rc = fn(ctypes.byref(self.geom), _ptr(fpost), _ptr(self.flags),
                self.inlet_u, z0, z1)
        if rc:
            raise RuntimeError(f"orc_open_pass failed ({rc})")

    def step(self, fpre, fpost):
        """Fused update only (the reference's KernelPlan.step)."""
        self.step_range(fpre, fpost, 0, self.geom.nz)

    def open_pass(self, fpost):
        self.open_pass_range(fpost, 0, self.geom.nz)

    def macro(self, f):
        """(rho, ux, uy, uz) as float64 a[x, y, z] grids, all cells."""
        self._check(f)
        g = self.geom
        n = g.nx * g.ny * g.nz
        out = [np.empty(n, dtype=np.float64) for _ in range(4)]
        fn = getattr(lib(), f"orc_macro_{_suffix(f.dtype)}")
        fn(ctypes.byref(g), _ptr(f), *[_ptr(o) for o in out])
        return tuple(o.reshape(g.nz, g.ny, g.nx).transpose(2, 1, 0) for o in out)

    def diagnostics(self, f):
        self._check(f)
        out = np.empty(8, dtype=np.float64)
        fn = getattr(lib(), f"orc_diag_{_suffix(f.dtype)}")
        fn(ctypes.byref(self.geom), _ptr(f), _ptr(self.flags), _ptr(out))
        keys = ("mass", "px", "py", "pz", "kinetic_energy", "max_u",
                "nonfinite", "fluid_cells")
        return dict(zip(keys, out.tolist()))


class CpuOracle(_Base):
    """Whole periodic domain, dense `(19, nx*ny*nz)` blocks, x fastest."""

    def __init__(self, nx, ny, nz, flags, omega, wall_u=(0.0, 0.0, 0.0),
                 inlet_u=0.0, threads=1, compute=None):
        flags = np.ascontiguousarray(flags, dtype=np.uint8).reshape(-1)
        n = nx * ny * nz
        if flags.size != n:
            raise ValueError("flag array does not match the grid")
        geom = Geom(nx, ny, nz, nx, nx * ny, n, 0, nz - 1, 0)
        super().__init__(geom, flags, omega, wall_u, inlet_u, threads, compute)

    def run(self, fpre, fpost, steps):
        """`steps` x (fused update, open-boundary pass, swap); returns the
        buffer holding the newest populations (engine.py:244-249)."""
        for _ in range(steps):
            self.step(fpre, fpost)
            self.open_pass(fpost)
            fpre, fpost = fpost, fpre
        return fpre


class SlabOracle(_Base):
    """One z-slab: blocks `(19, nz+2, ny, xp)`, halo planes at storage index
    0 and nz+1 supply the pulls from lz = -1 and lz = nz."""

    def __init__(self, nx, ny, nz, xp, flags, omega, wall_u=(0.0, 0.0, 0.0),
                 inlet_u=0.0, threads=1, compute=None):
        flags = np.ascontiguousarray(flags, dtype=np.uint8)
        if flags.shape != (nz + 2, ny, xp):
            raise ValueError("slab flags must have shape (nz+2, ny, xp)")
        geom = Geom(nx, ny, nz, xp, ny * xp, (nz + 2) * ny * xp, 1, 0, nz + 1)
        super().__init__(geom, flags, omega, wall_u, inlet_u, threads, compute)


def equilibrium(rho, ux, uy, uz, dtype):
    """Equilibrium in the COMPUTE dtype of a storage dtype (float32 for
    float16 storage)."""
    cdtype = np.float32 if np.dtype(dtype) == np.float16 else dtype
    out = np.empty(19, dtype=cdtype)
    getattr(lib(), f"orc_equilibrium_{_suffix(dtype)}")(
        float(rho), float(ux), float(uy), float(uz), _ptr(out))
    return out
