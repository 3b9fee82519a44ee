"""Generate the golden fixtures in this directory from the REAL reference.

Run in the build container only (it imports the unmodified reference from
/root/reference, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Everything written here is an output of the reference's own code
(`lb2d`, numba backend, and its independent test oracle
`pkg/tests/reference.py`) on deterministic inputs; the tests compare the
D3Q19 oracle and the CUDA path against these files through the
z-projection bridge (a z-invariant, z-periodic D3Q19 state summed over c_z
is a D2Q9 state).  Nothing here is hand-edited.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, REF)

os.environ["LB2D_BACKEND"] = "numba"

from lb2d import boundaries, cases, engine, kernels, lattice  # noqa: E402
from lb2d.fields import Layout, PopulationField, Precision  # noqa: E402
from tests.reference import ref_step  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 20240917  # the reference's fixture seed (pkg/tests/conftest.py:7)


def run_case(spec, precision, steps):
    state = cases.init(spec, precision, Layout.ROW)
    f0 = state.f_pre.data.copy()
    engine.run(state, engine.RunConfig(steps=steps, precision=precision,
                                       layout=Layout.ROW))
    rho, ux, uy = state.macro()
    return dict(nx=spec.nx, ny=spec.ny, steps=steps, omega=state.params.omega,
                nu=state.params.nu, wall_u=np.array(state.wall_u),
                inlet_u=state.inlet_u, mask=state.mask.copy(),
                f0=f0, f=state.f_pre.data.copy(), rho=rho, ux=ux, uy=uy)


def kernel_geometries():
    # pkg/tests/test_kernels.py:25-33
    cavity = boundaries.cavity_mask(9, 7)
    cavity[4, 3] = boundaries.SOLID
    channel = boundaries.channel_mask(12, 8, boundaries.disk_cells(12, 8, 4, 4.0, 3.5))
    periodic = boundaries.open_mask(6, 6)
    return {"cavity": (cavity, (0.08, 0.0)),
            "channel": (channel, (0.0, 0.0)),
            "periodic": (periodic, (0.0, 0.0))}


def main():
    assert kernels.BACKEND == "numba", kernels.BACKEND
    out = {}

    # --- cases through the reference engine (D2Q9, ROW layout) -------------
    ldc = cases.CaseSpec("ldc", 24, 24, re=100.0, u0=0.1)
    for tag, prec in (("f64", Precision.DOUBLE), ("f32", Precision.SINGLE),
                      ("m2", Precision.MIXED2)):
        for k, v in run_case(ldc, prec, 100).items():
            out[f"ldc24_{tag}_{k}"] = v
    tgv = cases.CaseSpec("tgv", 16, 16, re=50.0, u0=0.04)
    for k, v in run_case(tgv, Precision.DOUBLE, 50).items():
        out[f"tgv16_f64_{k}"] = v
    vks = cases.CaseSpec("vks", 48, 32, re=60.0, u0=0.1)
    out["vks_diameter"] = vks.diameter
    out["vks_cyl"] = np.array([vks.cyl_x, vks.cyl_y])
    for k, v in run_case(vks, Precision.DOUBLE, 60).items():
        out[f"vks48_f64_{k}"] = v

    # --- one fused step on the reference's three kernel-test geometries ----
    rng = np.random.default_rng(SEED)
    for name, (grid, wall_u) in kernel_geometries().items():
        nx, ny = grid.shape
        f = PopulationField.alloc(nx, ny, Layout.ROW, np.float64)
        f.data[:] = rng.uniform(0.02, 1.0, size=f.data.shape)
        mask = boundaries.flatten_mask(grid, Layout.ROW)
        post = f.copy()
        kernels.KernelPlan(nx, ny, Layout.ROW, Precision.DOUBLE, mask, 1.41,
                           wall_u, backend="numba").step(f.data, post.data)
        fxy = np.stack([f.plane_xy(i) for i in range(9)], axis=-1)
        want = ref_step(fxy, grid, 1.41, wall_u=wall_u)
        out[f"k1_{name}_grid"] = grid
        out[f"k1_{name}_wall_u"] = np.array(wall_u)
        out[f"k1_{name}_f0"] = f.data.copy()
        out[f"k1_{name}_numba"] = post.data.copy()
        out[f"k1_{name}_refstep"] = want  # (nx, ny, 9), the independent oracle

    # --- known answers and geometry bytes ------------------------------------
    out["eq_rho1_u01"] = lattice.equilibrium(1.0, 0.1, 0.0)
    out["eq_rho12_u"] = lattice.equilibrium(1.2, 0.05, -0.07)
    out["omega_re1000"] = lattice.omega_from_reynolds(1000, 0.1, 100).omega
    out["omega_re6"] = lattice.omega_from_reynolds(6, 0.1, 10).omega
    out["mw_diag"] = boundaries.moving_wall_correction(0.0, 5, (0.1, 0.0))
    out["mw_axis"] = boundaries.moving_wall_correction(0.25, 1, (0.1, 0.0))
    out["mask_cavity_6x5"] = boundaries.cavity_mask(6, 5)
    out["mask_cavity_24"] = boundaries.cavity_mask(24, 24)
    out["mask_channel_8x6"] = boundaries.channel_mask(8, 6)
    out["mask_channel_disk"] = boundaries.channel_mask(
        16, 12, boundaries.disk_cells(16, 12, 4, 6.0, 6.0))
    out["disk_20"] = boundaries.disk_cells(20, 20, 6, 10.0, 10.0)
    out["disk_half"] = boundaries.disk_cells(16, 16, 5, 8.0, 7.5)
    out["tgv_fields_16"] = np.stack(cases.tgv_fields(16, 0.04, 0.01, 7.0))
    out["flags_codes"] = np.array([boundaries.FLUID, boundaries.SOLID,
                                   boundaries.MOVING_WALL, boundaries.INLET,
                                   boundaries.OUTLET], dtype=np.uint8)

    # wake analysis (cases.py:200-228) on a noisy, drifting two-tone series
    rs = np.random.default_rng(20240917)
    t = np.arange(3000, dtype=np.float64)
    series = (0.02 * np.sin(2 * np.pi * t / 173.0) + 0.004 * np.sin(2 * np.pi * t / 41.0)
              + 3e-6 * t + 0.002 * rs.standard_normal(t.size))
    out["strouhal_series"] = series
    out["strouhal_crossings"] = cases.zero_crossing_times(series)
    st, n = cases.strouhal(series, 16.0, 0.08, sample_every=2)
    out["strouhal_value"] = np.array([st, n], dtype=np.float64)

    path = os.path.join(HERE, "lb2d_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
