"""The in-place (AA pattern) update: one population block, same bits.

Arithmetic and operands are those of the two-buffer kernel, so after any
number of steps - odd or even, through the shifted representation and back
- the populations must equal the CPU oracle's bit for bit, and non-fluid
cells must be untouched."""

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import lattice as L
from paper_2409_16781_b200.fields import Layout, Precision

from .helpers import geometries3d, random_block

pytestmark = pytest.mark.gpu

PREC = {"f32": Precision.SINGLE, "f64": Precision.DOUBLE, "f16": Precision.MIXED1,
        "m2": Precision.MIXED2}
WALL_GEOMS = ["porous", "cavity", "cavity_oblique_lid", "cavity16", "periodic", "periodic8", "wide"]


def make(grid, prec, omega, wall_u):
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = grid.shape
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), omega, wall_u)
    orc = CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u,
                    compute=np.float64 if prec is Precision.MIXED2 else None)
    return plan, orc


@pytest.mark.parametrize("steps", [1, 2, 5, 8])
@pytest.mark.parametrize("tag", ["f64", "f32", "f16", "m2"])
@pytest.mark.parametrize("geom", WALL_GEOMS)
def test_inplace_equals_oracle_bitwise(geom, tag, steps, rng):
    grid, wall_u, _ = geometries3d()[geom]
    prec = PREC[tag]
    plan, orc = make(grid, prec, 1.45, wall_u)
    f = random_block(rng, grid.size, prec.storage)
    want = orc.run(f.copy(), f.copy(), steps)
    d = plan.alloc()
    plan.upload(f, d)
    plan.run_steps_inplace(d, steps)
    assert d.repr == steps % 2
    plan.normalize(d)
    assert d.repr == 0
    got = np.empty_like(f)
    plan.download(d, got)
    np.testing.assert_array_equal(got, want)


PACK_VARIANTS = {"f32": [1008, 1016, 1032, 2008, 2016], "f64": [1008, 1016, 1032],
                 "f16": [2008, 2016, 2032, 3008, 3016, 3032], "m2": [2008, 2016, 2032]}


@pytest.mark.parametrize("steps", [1, 2, 7])
@pytest.mark.parametrize("tag,variant", [(t, v) for t in PACK_VARIANTS for v in PACK_VARIANTS[t]])
@pytest.mark.parametrize("geom", ["porous", "cavity16", "periodic8", "wide"])
def test_inplace_pack_kernels_bitwise(geom, tag, variant, steps, rng):
    """The vectorised in-place kernels (aligned packs, the pack-boundary cell
    passed between lanes by a shuffle): ragged rows, walls inside and between
    packs, lanes outside the grid, periodic wrap at both row ends."""
    grid, wall_u, _ = geometries3d()[geom]
    prec = PREC[tag]
    plan, orc = make(grid, prec, 1.45, wall_u)
    plan.set_variant(variant)
    f = random_block(rng, grid.size, prec.storage)
    want = orc.run(f.copy(), f.copy(), steps)
    d = plan.alloc()
    plan.upload(f, d)
    plan.run_steps_inplace(d, steps)
    plan.normalize(d)
    got = np.empty_like(f)
    plan.download(d, got)
    np.testing.assert_array_equal(got, want)


def test_split_runs_and_normalize_in_the_middle(rng):
    grid, wall_u, _ = geometries3d()["cavity16"]
    plan, orc = make(grid, Precision.SINGLE, 1.7, wall_u)
    f = random_block(rng, grid.size, np.float32)
    want = orc.run(f.copy(), f.copy(), 9)
    d = plan.alloc()
    plan.upload(f, d)
    plan.run_steps_inplace(d, 3)     # ends shifted
    plan.normalize(d)                # back to normal without stepping
    mid = np.empty_like(f)
    plan.download(d, mid)
    np.testing.assert_array_equal(mid, orc.run(f.copy(), f.copy(), 3))
    plan.normalize(d)                # no-op in the normal representation
    plan.run_steps_inplace(d, 1)
    plan.run_steps_inplace(d, 5)     # continues from the shifted representation
    plan.normalize(d)
    got = np.empty_like(f)
    plan.download(d, got)
    np.testing.assert_array_equal(got, want)
    # diagnostics on the normalised block equal the two-buffer path's
    a, b = plan.alloc(), plan.alloc()
    plan.upload(f, a)
    plan.upload(f, b)
    newest, _, _ = plan.run_steps(a, b, 9)
    assert plan.diagnostics(d) == plan.diagnostics(newest)


@pytest.mark.parametrize("steps", [1, 2, 7])
@pytest.mark.parametrize("tag,variant", [("f32", 1008), ("f32", 1016), ("f64", 1008), ("f64", 1032),
                                         ("f16", 2008), ("f16", 3016)])
@pytest.mark.parametrize("geom", ["channel40", "duct", "channel"])
def test_inplace_open_boundaries_bitwise(geom, tag, variant, steps, rng):
    """Inlet / outlet cells in place: with the pack kernels every non-wall cell
    takes part in the exchange of slots - inlet cells' new state is the
    constant equilibrium, outlet cells copy their x-1 neighbour inside the
    pack - and the result equals step + open-boundary pass of the oracle."""
    from paper_2409_16781_b200.kernels import KernelPlan
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    prec = PREC[tag]
    # ("channel" has nx = 14: the four-cell packs end in a pack of two cells + padding,
    # which holds the outlet cell and the fluid cell it copies)
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), 1.3, wall_u,
                      inlet_u=inlet_u)
    plan.set_variant(variant)
    orc = CpuOracle(nx, ny, nz, B.flatten_mask(grid), 1.3, wall_u, inlet_u)
    f = random_block(rng, grid.size, prec.storage)
    want = orc.run(f.copy(), f.copy(), steps)
    d = plan.alloc()
    plan.upload(f, d)
    plan.run_steps_inplace(d, steps)
    plan.normalize(d)
    got = np.empty_like(f)
    plan.download(d, got)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("geom", ["open_chain", "open_unfusable"])
def test_inplace_refuses_outlets_it_cannot_serve_inside_a_pack(geom):
    from paper_2409_16781_b200.kernels import KernelPlan
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE, B.flatten_mask(grid), 1.0,
                      wall_u, inlet_u=inlet_u)
    plan.set_variant(1008)
    with pytest.raises(ValueError, match="walls only"):
        plan.run_steps_inplace(plan.alloc(zero=True), 1)


def test_open_boundaries_are_rejected(rng):
    grid, wall_u, inlet_u = geometries3d()["channel40"]
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = grid.shape
    plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE, B.flatten_mask(grid), 1.0,
                      wall_u, inlet_u=inlet_u)
    d = plan.alloc(zero=True)
    with pytest.raises(ValueError, match="walls only"):
        plan.run_steps_inplace(d, 1)
    from paper_2409_16781_b200 import cases, engine
    state = cases.init(cases.CaseSpec("vks", 48, 32, 8), Precision.SINGLE)
    with pytest.raises(ValueError, match="walls only"):
        engine.run(state, engine.RunConfig(steps=1, inplace=True))


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_engine_run_inplace_equals_two_buffer_run(tag):
    from paper_2409_16781_b200 import cases, engine
    prec = PREC[tag]
    spec = cases.CaseSpec("ldc", 40, 36, 28, re=100.0, u0=0.1)
    a = cases.init(spec, prec)
    b = cases.init(spec, prec)
    seen = []
    ra = engine.run(a, engine.RunConfig(steps=31, precision=prec, output_every=10),
                    on_output=lambda st: seen.append(st.t), probe=(20, 30, 14))
    rb = engine.run(b, engine.RunConfig(steps=31, precision=prec, output_every=10, inplace=True),
                    probe=(20, 30, 14))
    assert seen == [10, 20, 30] and a.t == b.t == 31
    np.testing.assert_array_equal(a.f_pre.data, b.f_pre.data)
    np.testing.assert_array_equal(ra.probe_samples, rb.probe_samples)
    for x, y in zip(a.macro(), b.macro()):
        np.testing.assert_array_equal(x, y)


def test_ldc_1024_cubed_fp32_on_one_gpu():
    """BASELINE configs[3]'s grid on ONE B200: 1024^3 fp32 needs 81.7 GB per
    block; two blocks plus tables would not leave room, one block does.
    Properties at full size: mass conservation in the closed box, finite
    fields, walls untouched, the lid drags fluid along +x."""
    import torch
    from paper_2409_16781_b200.kernels import KernelPlan
    from paper_2409_16781_b200.lattice import omega_from_reynolds
    n = 1024
    free, _ = torch.cuda.mem_get_info()
    if free < 100e9:
        pytest.skip("needs ~95 GB of free device memory")
    omega = omega_from_reynolds(1000.0, 0.1, n).omega
    flags = B.flatten_mask(B.cavity_mask(n, n, n))
    plan = KernelPlan(n, n, n, Layout.ROW, Precision.SINGLE, flags, omega, (0.1, 0.0, 0.0))
    del flags
    d = plan.alloc()
    for q in range(19):
        d.tensor[q].fill_(float(np.float32(L.W[q])))
    d0 = plan.diagnostics(d)
    assert d0["fluid_cells"] == (n - 2) ** 3
    ms = plan.run_steps_inplace(d, 6, timed=True)
    plan.normalize(d)
    d1 = plan.diagnostics(d)
    assert d1["nonfinite"] == 0
    assert abs(d1["mass"] - d0["mass"]) <= 2e-6 * d0["mass"]
    assert 0.0 < d1["max_u"] < 0.2 and d1["px"] > 0.0
    wall = d.tensor[:, 1:-1, 0, :n]
    assert all(bool((wall[q] == float(np.float32(L.W[q]))).all()) for q in range(19))
    print(f"1024^3 fp32 in place: {n ** 3 * 6 / ms / 1e3:.0f} MLUPS")


def test_engine_run_inplace_channel_equals_two_buffer_run():
    """engine.run(inplace=True) on a channel with inlet, outlet and obstacle
    (nx = 128: the pack kernels serve the open boundaries inside the step)."""
    from paper_2409_16781_b200 import cases, engine
    spec = cases.CaseSpec("vks", 128, 48, 12, re=100.0, u0=0.08)
    a = cases.init(spec, Precision.SINGLE)
    b = cases.init(spec, Precision.SINGLE)
    engine.run(a, engine.RunConfig(steps=23))
    engine.run(b, engine.RunConfig(steps=23, inplace=True))
    np.testing.assert_array_equal(a.f_pre.data, b.f_pre.data)
    orc = CpuOracle(128, 48, 12, a.mask, a.params.omega, inlet_u=a.inlet_u, threads=8)
    f0 = cases.init(spec, Precision.SINGLE).f_pre.data
    np.testing.assert_array_equal(a.f_pre.data, orc.run(f0.copy(), f0.copy(), 23))


def _row_block_grids():
    """Rows that exactly fill a block of 1, 2 or 4 warps (the periodic wrap then
    closes inside the block), rows that do not, walls inside and between packs,
    inlet / outlet faces."""
    out = {}
    for nx, ny, nz in ((128, 6, 4), (256, 5, 3), (512, 4, 3), (72, 4, 3), (200, 5, 3)):
        g = B.open_mask(nx, ny, nz)
        u = np.random.default_rng(nx).random(g.shape)
        g[u < 0.03] = B.SOLID
        g[u > 0.985] = B.MOVING_WALL
        out[f"periodic{nx}"] = (g, (0.03, -0.02, 0.04), 0.0)
    cav = B.cavity_mask(256, 8, 5)
    cav[100:104, 3:5, 2] = B.SOLID
    out["cavity256"] = (cav, (0.06, 0.0, 0.0), 0.0)
    out["channel128"] = (B.channel_mask(128, 8, 5, B.sphere_cells(128, 8, 5, 4, 30.0, 4.0, 2.5)),
                         (0.0, 0.0, 0.0), 0.05)
    return out


@pytest.mark.parametrize("tag,variant", [("f32", 1016), ("f64", 1016), ("f16", 2016), ("m2", 2016),
                                         ("f32", 2016)])
@pytest.mark.parametrize("geom", list(_row_block_grids()))
def test_inplace_row_block_layout_never_changes_bits(geom, tag, variant, rng):
    """mlb_plan_set_inplace_layout(1): the pull half's warps sit side by side in
    x and hand the value that crosses a warp boundary through shared memory.  A
    thread layout, like the reference's tiles (test_kernels.py:107-126): same
    bits as the oracle, odd and even step counts."""
    from paper_2409_16781_b200.kernels import KernelPlan
    grid, wall_u, inlet_u = _row_block_grids()[geom]
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    flags = B.flatten_mask(grid)
    f = random_block(rng, grid.size, prec.storage)
    orc = CpuOracle(nx, ny, nz, flags, 1.5, wall_u, inlet_u,
                    compute=np.float64 if prec is Precision.MIXED2 else None)
    for steps in (1, 4):
        want = orc.run(f.copy(), f.copy(), steps)
        plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, flags, 1.5, wall_u, inlet_u=inlet_u)
        plan.set_variant(variant)
        plan.set_inplace_layout(1)
        d = plan.alloc()
        plan.upload(f, d)
        plan.run_steps_inplace(d, steps)
        plan.normalize(d)
        got = np.empty_like(f)
        plan.download(d, got)
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("tag,variant", [("f32", 1008), ("f32", 1016), ("f16", 2016), ("m2", 2016),
                                         ("f64", 1016)])
@pytest.mark.parametrize("shape", [(13, 6, 5), (15, 5, 4), (101, 4, 3), (131, 9, 3), (259, 4, 3)])
def test_inplace_pack_kernels_on_ragged_rows(shape, tag, variant, layout, rng):
    """Rows the pack does not divide, in place: the last pack holds real cells +
    padding, and the cell at x = nx-1 pulls from / writes to cell 0 of the row
    across the periodic wrap.  Periodic box with scattered walls and a cavity,
    both thread layouts of the pull half, odd and even step counts."""
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = shape
    prec = PREC[tag]
    for kind in ("periodic", "cavity"):
        grid = B.open_mask(nx, ny, nz) if kind == "periodic" else B.cavity_mask(nx, ny, nz)
        u = np.random.default_rng(nx + 1).random(grid.shape)
        grid[(u < 0.05) & (grid == B.FLUID)] = B.SOLID
        grid[(u > 0.97) & (grid == B.FLUID)] = B.MOVING_WALL
        flags = B.flatten_mask(grid)
        wall_u = (0.04, -0.02, 0.03)
        f = random_block(rng, grid.size, prec.storage)
        orc = CpuOracle(nx, ny, nz, flags, 1.6, wall_u,
                        compute=np.float64 if prec is Precision.MIXED2 else None)
        for steps in (1, 4):
            want = orc.run(f.copy(), f.copy(), steps)
            plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, flags, 1.6, wall_u)
            plan.set_variant(variant)
            plan.set_inplace_layout(layout)
            d = plan.alloc()
            plan.upload(f, d)
            plan.run_steps_inplace(d, steps)
            plan.normalize(d)
            got = np.empty_like(f)
            plan.download(d, got)
            np.testing.assert_array_equal(got, want)
