"""ctypes binding of libmlb_d3q19.so (include/mlb.h).

The library is built in-tree by csrc/Makefile (`__graft_entry__.build()`);
there is no fallback: if it is missing, importing the compute path raises.
Error codes map to the exception types the reference raises at the same
points (kernels.py:416-427, engine.py:184-187): MLB_EINVAL and
MLB_EUNSUPPORTED -> ValueError, MLB_ENOMEM -> MemoryError, MLB_ECUDA ->
RuntimeError.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# (MLB_LIB_PATH: A/B experiments with a second build, tools/ only)
LIB_PATH = os.environ.get("MLB_LIB_PATH") or os.path.join(_HERE, "libmlb_d3q19.so")
ABI_VERSION = 2

MLB_F32, MLB_F64, MLB_F16, MLB_F32C64 = 0, 1, 2, 3
IPC_HANDLE_BYTES = 64
MLB_Z_PERIODIC, MLB_Z_HALO = 0, 1
MLB_OK, MLB_EINVAL, MLB_ECUDA, MLB_ENOMEM, MLB_EUNSUPPORTED = 0, 1, 2, 3, 4

#: every symbol include/mlb.h declares; tests check the .so exports them all
SYMBOLS = (
    "mlb_last_error", "mlb_abi_version", "mlb_build_id", "mlb_launch_count", "mlb_trim", "mlb_layout_query",
    "mlb_plan_create", "mlb_plan_destroy", "mlb_plan_get_layout",
    "mlb_plan_set_physics", "mlb_plan_set_variant", "mlb_plan_set_passthrough",
    "mlb_plan_set_prefetch",
    "mlb_plan_kernel_name", "mlb_plan_set_flags",
    "mlb_plan_get_flags", "mlb_plan_geometry_stats", "mlb_upload", "mlb_download", "mlb_step",
    "mlb_step_range", "mlb_step_open_range", "mlb_open_pass", "mlb_open_pass_range",
    "mlb_run_steps",
    "mlb_run_steps_inplace", "mlb_inplace_normalize",
    "mlb_step_inplace_range", "mlb_inplace_swap_slab",
    "mlb_halo_copy", "mlb_halo_push", "mlb_step_push_range",
    "mlb_ipc_export", "mlb_ipc_open", "mlb_ipc_close",
    "mlb_signal_create", "mlb_signal_destroy", "mlb_signal_post", "mlb_signal_wait",
    "mlb_signal_wait_kind", "mlb_signal_read", "mlb_macro", "mlb_diagnostics", "mlb_probe",
    "mlb_step_host",
    "mlb_block_alloc", "mlb_block_free", "mlb_plan_set_graph",
    "mlb_slab_run_steps", "mlb_slab_run_steps_inplace", "mlb_run_steps_host",
    "mlb_plan_set_inplace_layout",
)


class Layout(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("itemsize", ctypes.c_int32), ("xp", ctypes.c_int64),
                ("plane", ctypes.c_int64), ("pop", ctypes.c_int64),
                ("total", ctypes.c_int64), ("bytes", ctypes.c_int64)]


class Ring(ctypes.Structure):
    """mlb_ring (include/mlb.h): one rank's view of the z-slab ring."""
    _fields_ = [("below", ctypes.c_void_p * 2), ("above", ctypes.c_void_p * 2),
                ("nz_below", ctypes.c_int32), ("nz_above", ctypes.c_int32),
                ("post_below", ctypes.c_void_p), ("post_above", ctypes.c_void_p),
                ("wait_below", ctypes.c_void_p), ("wait_above", ctypes.c_void_p),
                ("t", ctypes.c_uint32), ("wait_mode", ctypes.c_int32),
                ("overlap", ctypes.c_int32)]


_lib = None


def lib():
    """The loaded library.  Raises RuntimeError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built "
            f"(run `python -c 'import __graft_entry__ as g; g.build()'` or "
            f"`make -C paper_2409_16781_b200/csrc`).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    dp3 = ctypes.POINTER(ctypes.c_double)
    sig = {
        "mlb_last_error": (ctypes.c_char_p, []),
        "mlb_abi_version": (i, []),
        "mlb_build_id": (ctypes.c_char_p, []),
        "mlb_launch_count": (ctypes.c_int64, []),
        "mlb_trim": (i, []),
        "mlb_layout_query": (i, [i, i, i, i, ctypes.POINTER(Layout)]),
        "mlb_plan_create": (i, [ctypes.POINTER(vp), i, i, i, i, d, dp3, d, i, i]),
        "mlb_plan_destroy": (i, [vp]),
        "mlb_plan_get_layout": (i, [vp, ctypes.POINTER(Layout)]),
        "mlb_plan_set_physics": (i, [vp, d, dp3, d]),
        "mlb_plan_set_variant": (i, [vp, i]),
        "mlb_plan_set_passthrough": (i, [vp, i]),
        "mlb_plan_set_prefetch": (i, [vp, ctypes.c_longlong]),
        "mlb_plan_kernel_name": (ctypes.c_char_p, [vp]),
        "mlb_plan_set_flags": (i, [vp, vp, vp, vp]),
        "mlb_plan_get_flags": (i, [vp, vp]),
        "mlb_plan_geometry_stats": (i, [vp, ctypes.POINTER(ctypes.c_int64)]),
        "mlb_upload": (i, [vp, vp, vp, vp]),
        "mlb_download": (i, [vp, vp, vp, vp]),
        "mlb_step": (i, [vp, vp, vp, vp]),
        "mlb_step_range": (i, [vp, vp, vp, i, i, vp]),
        "mlb_step_open_range": (i, [vp, vp, vp, i, i, vp]),
        "mlb_open_pass": (i, [vp, vp, vp]),
        "mlb_open_pass_range": (i, [vp, vp, i, i, vp]),
        "mlb_run_steps": (i, [vp, vp, vp, i, vp, ctypes.POINTER(ctypes.c_float)]),
        "mlb_run_steps_inplace": (i, [vp, vp, i, ctypes.POINTER(ctypes.c_int), vp,
                                      ctypes.POINTER(ctypes.c_float)]),
        "mlb_inplace_normalize": (i, [vp, vp, ctypes.POINTER(ctypes.c_int), vp]),
        "mlb_step_inplace_range": (i, [vp, vp, i, i, i, vp, i, vp, i, vp]),
        "mlb_inplace_swap_slab": (i, [vp, vp, vp, i, vp]),
        "mlb_halo_copy": (i, [vp, vp, vp, i, i, vp]),
        "mlb_halo_push": (i, [vp, vp, vp, i, i, vp]),
        "mlb_step_push_range": (i, [vp, vp, vp, i, i, vp, i, vp, i, vp]),
        "mlb_ipc_export": (i, [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
        "mlb_ipc_open": (i, [i, ctypes.c_char_p, ctypes.POINTER(vp)]),
        "mlb_ipc_close": (i, [vp]),
        "mlb_signal_create": (i, [i, ctypes.POINTER(vp)]),
        "mlb_signal_destroy": (i, [vp]),
        "mlb_signal_post": (i, [vp, ctypes.c_uint32, vp]),
        "mlb_signal_wait": (i, [vp, ctypes.c_uint32, i, vp]),
        "mlb_signal_wait_kind": (i, []),
        "mlb_signal_read": (i, [vp, ctypes.POINTER(ctypes.c_uint32)]),
        "mlb_macro": (i, [vp, vp, vp, vp, vp, vp, vp]),
        "mlb_diagnostics": (i, [vp, vp, dp3, vp]),
        "mlb_probe": (i, [vp, vp, i, i, i, vp, vp]),
        "mlb_step_host": (i, [vp, vp, vp, vp, vp, vp]),
        "mlb_block_alloc": (i, [i, ctypes.c_int64, ctypes.POINTER(vp)]),
        "mlb_block_free": (i, [vp]),
        "mlb_plan_set_graph": (i, [vp, i]),
        "mlb_plan_set_inplace_layout": (i, [vp, i]),
        "mlb_run_steps_host": (i, [vp, vp, vp, vp, vp, i, i, vp, vp,
                                   ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i)]),
        "mlb_slab_run_steps": (i, [vp, vp, vp, i, ctypes.POINTER(Ring), vp, vp,
                                   ctypes.POINTER(d)]),
        "mlb_slab_run_steps_inplace": (i, [vp, vp, i, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(Ring), vp, vp, ctypes.POINTER(d)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.mlb_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB_PATH}: ABI version {L.mlb_abi_version()} "
                           f"!= expected {ABI_VERSION}; rebuild the extension")
    _lib = L
    return L


def check(rc):
    """Raise the Python exception matching a non-zero MLB_E* return code."""
    if rc == MLB_OK:
        return
    msg = lib().mlb_last_error().decode("utf-8", "replace")
    if rc in (MLB_EINVAL, MLB_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == MLB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def build_id():
    """Hash of the sources the loaded library was built from."""
    return lib().mlb_build_id().decode()


def launch_count():
    return int(lib().mlb_launch_count())
