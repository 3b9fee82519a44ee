"""B200-native D3Q19 time-step loop behind the miniLB (`lb2d`) plugin API.

Host modules (`lattice`, `fields`, `boundaries`, `perfport`) are pure numpy
and import anywhere.  `kernels`, `engine` and `cases` drive the CUDA path
through libmlb_d3q19.so (include/mlb.h) and need torch; they are imported
lazily so that the host modules stay usable on a machine without a GPU.
"""

from . import boundaries, fields, lattice, perfport  # noqa: F401

__all__ = ["boundaries", "fields", "lattice", "perfport", "kernels", "engine",
           "cases", "slab", "io"]


def __getattr__(name):
    if name in ("kernels", "engine", "cases", "slab", "io", "_cabi"):
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
