"""File surfaces of the hot path: VTK snapshots.

3-D counterpart of the reference's `write_vtk`
(/root/reference/pkg/src/lb2d/io.py:21-53): legacy ASCII structured points,
one density scalar and one velocity vector per cell, x fastest, values
written as float32 with shortest-round-trip formatting (`%.9g`) so identical
states always serialise to identical bytes.  For nz = 1 the file is byte for
byte what the reference writes.  The fields come from `state.macro()`, i.e.
from the CUDA macro kernel.  The reference's CSV / argparse surfaces are out
of scope.
"""

import numpy as np


def _column(a):
    """float64 a[x, y, z] -> list of '%.9g' strings of float32(a), x fastest."""
    flat = np.ascontiguousarray(a.astype(np.float32).transpose(2, 1, 0)).reshape(-1)
    return ["%.9g" % float(v) for v in flat]


def write_vtk(path, state, fields=None):
    """Write one legacy ASCII snapshot of density and velocity.

    `fields` = (rho, ux, uy, uz) as a[x, y, z] grids overrides
    `state.macro()` (used by tests that have no GPU).
    """
    rho, ux, uy, uz = fields if fields is not None else state.macro()
    nx, ny, nz = state.nx, state.ny, state.nz
    lines = [
        "# vtk DataFile Version 3.0",
        f"miniLB t={state.t}",
        "ASCII",
        "DATASET STRUCTURED_POINTS",
        f"DIMENSIONS {nx} {ny} {nz}",
        "ORIGIN 0 0 0",
        "SPACING 1 1 1",
        f"POINT_DATA {nx * ny * nz}",
        "SCALARS density float 1",
        "LOOKUP_TABLE default",
    ]
    lines.extend(_column(rho))
    lines.append("VECTORS velocity float")
    lines.extend(f"{a} {b} {c}" for a, b, c in zip(_column(ux), _column(uy), _column(uz)))
    with open(path, "w", newline="\n") as fh:
        fh.write("\n".join(lines))
        fh.write("\n")
