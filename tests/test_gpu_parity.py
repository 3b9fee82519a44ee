"""GPU parity: the CUDA path, called through the C ABI, against the CPU
oracle on identical inputs.  The bar for populations and macroscopic fields
is BIT-EXACT (stronger than the 1e-12 / 1e-5 relative tolerance the
north star allows): both sides perform the same IEEE operations in the
same order, neither contracts multiplies and adds."""

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from oracle.ref3d import ref3d_open_pass, ref3d_step
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision

from .helpers import (extrude_mask, from_xyzq, geometries3d, lift_2d,
                      project_2d, random_block, to_xyzq)

pytestmark = pytest.mark.gpu

PREC = {"f32": Precision.SINGLE, "f64": Precision.DOUBLE, "f16": Precision.MIXED1,
        "m2": Precision.MIXED2}
VARIANTS = {"f32": [32, 64, 128, 256, 512, 1008, 1016, 1032, 2008, 2016, 2032],
            "f64": [32, 64, 128, 256, 512, 1008, 1016, 1032],
            "f16": [32, 128, 512, 2008, 2016, 2032, 3008, 3016, 3032],
            "m2": [32, 128, 512, 2008, 2016, 2032]}


def make_plan(grid, prec, omega, wall_u, inlet_u=0.0, **kw):
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = grid.shape
    return KernelPlan(nx, ny, nz, Layout.ROW, prec, B.flatten_mask(grid), omega,
                      wall_u, inlet_u=inlet_u, **kw)


def make_oracle(grid, omega, wall_u, inlet_u=0.0, prec=None):
    nx, ny, nz = grid.shape
    # the oracle computes in the storage dtype's own compute type unless told
    # otherwise: MIXED2 is float storage with double arithmetic
    compute = np.float64 if prec is Precision.MIXED2 else None
    return CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u, compute=compute)


@pytest.mark.parametrize("tag", ["f64", "f32", "f16", "m2"])
@pytest.mark.parametrize("geom", list(geometries3d()))
def test_one_step_bitwise(geom, tag, rng):
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = PREC[tag]
    n = grid.size
    f = random_block(rng, n, prec.storage)
    post0 = random_block(rng, n, prec.storage)  # never-written cells must survive
    omega = 1.41
    want = post0.copy()
    make_oracle(grid, omega, wall_u, inlet_u, prec).step(f, want)
    got = post0.copy()
    make_plan(grid, prec, omega, wall_u, inlet_u).step(f, got)  # host-block call
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("geom", ["cavity", "channel", "periodic"])
def test_one_step_matches_naive_oracle(geom, rng):
    # the independent explicit-loop oracle, the reference's own tolerance
    # for this check (test_kernels.py:61)
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny, nz = grid.shape
    f = random_block(rng, grid.size, np.float64)
    got = f.copy()
    make_plan(grid, Precision.DOUBLE, 1.41, wall_u, inlet_u).step(f, got)
    want = ref3d_step(to_xyzq(f, nx, ny, nz), grid, 1.41, wall_u)
    np.testing.assert_allclose(to_xyzq(got, nx, ny, nz), want, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("tag", ["f64", "f32", "f16", "m2"])
@pytest.mark.parametrize("geom", list(geometries3d()))
def test_multi_step_with_open_pass_bitwise(geom, tag, rng):
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = PREC[tag]
    f = random_block(rng, grid.size, prec.storage)
    omega, steps = 0.9, 7
    a, b = f.copy(), f.copy()
    want = make_oracle(grid, omega, wall_u, inlet_u, prec).run(a, b, steps)
    plan = make_plan(grid, prec, omega, wall_u, inlet_u)
    da, db = plan.alloc(), plan.alloc()
    plan.upload(f, da)
    plan.upload(f, db)
    newest, _, _ = plan.run_steps(da, db, steps)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want)


VEC_GEOMS = ["cavity16", "channel40", "periodic8", "wide", "duct", "open_chain", "open_unfusable",
             "porous"]


def test_pattern_dictionary_and_escape_cells():
    """The kernels read one index byte per cell into a dictionary of distinct
    wall-link patterns; geometries with more than 254 patterns send the
    overflow cells to full-width class words.  Both paths must report the
    reference's flag bytes exactly."""
    g = geometries3d()
    for name, escapes in (("cavity", False), ("channel40", False), ("porous", True)):
        grid, wall_u, inlet_u = g[name]
        plan = make_plan(grid, Precision.SINGLE, 1.0, wall_u, inlet_u)
        kinds, esc = plan.geometry_stats()
        assert 1 <= kinds <= 255
        assert (esc > 0) == escapes, (name, kinds, esc)
        np.testing.assert_array_equal(plan.device_flags(), B.flatten_mask(grid))


@pytest.mark.parametrize("passthrough", [False, True])
@pytest.mark.parametrize("tag,variant", [(t, v) for t in VARIANTS for v in VARIANTS[t]])
@pytest.mark.parametrize("geom", VEC_GEOMS)
def test_kernel_variants_never_change_bits(geom, tag, variant, passthrough, rng):
    """Block shape, vectorisation and the store mode are pure performance
    knobs (test_kernels.py:107-126): every variant, same bits as the oracle.
    Strict mode must preserve arbitrary never-written cells of the second
    buffer; pass-through mode is exercised under its precondition (the two
    buffers agree on non-fluid cells)."""
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = PREC[tag]
    f = random_block(rng, grid.size, prec.storage)
    sentinel = random_block(rng, grid.size, prec.storage)
    if passthrough:
        non_fluid = B.flatten_mask(grid) != B.FLUID
        sentinel[:, non_fluid] = f[:, non_fluid]
    omega, steps = 1.6, 3
    a, b = f.copy(), sentinel.copy()
    orc = make_oracle(grid, omega, wall_u, inlet_u, prec)
    want = orc.run(a, b, steps)
    plan = make_plan(grid, prec, omega, wall_u, inlet_u)
    plan.set_variant(variant)
    if passthrough and geom.startswith("open_"):
        # chained outlet cells: the reference's result depends on the stale
        # content of a never-written cell, so pass-through must be refused
        with pytest.raises(ValueError, match="outlet"):
            plan.set_passthrough(True)
        return
    plan.set_passthrough(passthrough)
    da, db = plan.alloc(), plan.alloc()
    plan.upload(f, da)
    plan.upload(sentinel, db)
    newest, _, _ = plan.run_steps(da, db, steps)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("cells", [0, 5, "row+1", "plane", "2planes+3rows", 10 ** 9, -1])
@pytest.mark.parametrize("tag", ["f32", "f64", "f16", "m2"])
@pytest.mark.parametrize("geom", ["cavity16", "channel40", "periodic8", "wide"])
def test_prefetch_distance_never_changes_bits(geom, tag, cells, rng):
    """The L2 prefetch of the pack kernels (mlb_plan_set_prefetch) is a pure
    performance knob like the reference's tile shape (test_kernels.py:107-126):
    any distance - off, inside a row, across rows and planes, beyond the
    domain, auto - same bits as the oracle, two blocks and in place."""
    grid, wall_u, inlet_u = geometries3d()[geom]
    nx, ny = grid.shape[0], grid.shape[1]
    cells = {"row+1": nx + 1, "plane": nx * ny, "2planes+3rows": 2 * nx * ny + 3 * nx}.get(cells, cells)
    prec = PREC[tag]
    f = random_block(rng, grid.size, prec.storage)
    want = make_oracle(grid, 1.6, wall_u, inlet_u, prec).run(f.copy(), f.copy(), 4)
    plan = make_plan(grid, prec, 1.6, wall_u, inlet_u)
    plan.set_variant({"f32": 1016, "f64": 1016, "f16": 2008, "m2": 2016}[tag])
    plan.set_prefetch(cells)
    plan.set_passthrough(True)
    a, b = plan.alloc(), plan.alloc()
    plan.upload(f, a)
    plan.upload(f, b)
    newest, _, _ = plan.run_steps(a, b, 4)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want)
    c = plan.alloc()
    plan.upload(f, c)
    plan.run_steps_inplace(c, 4)
    plan.normalize(c)
    plan.download(c, got)
    np.testing.assert_array_equal(got, want)


def test_prefetch_distance_is_validated():
    grid, wall_u, inlet_u = geometries3d()["cavity16"]
    plan = make_plan(grid, Precision.SINGLE, 1.0, wall_u, inlet_u)
    with pytest.raises(ValueError, match="prefetch"):
        plan.set_prefetch(-2)


@pytest.mark.parametrize("tag,variant", [("f32", 2008), ("f32", 2016), ("f64", 1008), ("m2", 2032),
                                         ("f16", 3016)])
def test_two_cell_packs_on_rows_that_four_does_not_divide(tag, variant, rng):
    """nx = 14: even, not a multiple of 4 - the 8-byte (fp32, mixed2), 16-byte
    (fp64) and 4-byte (fp16) packs of two cells serve it, two blocks and in
    place, inlet / outlet cells included."""
    grid, wall_u, inlet_u = geometries3d()["channel"]
    assert grid.shape[0] % 4 == 2
    prec = PREC[tag]
    f = random_block(rng, grid.size, prec.storage)
    want = make_oracle(grid, 1.7, wall_u, inlet_u, prec).run(f.copy(), f.copy(), 5)
    plan = make_plan(grid, prec, 1.7, wall_u, inlet_u)
    plan.set_variant(variant)
    plan.set_passthrough(True)
    a, b = plan.alloc(), plan.alloc()
    plan.upload(f, a)
    plan.upload(f, b)
    newest, _, _ = plan.run_steps(a, b, 5)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want)
    c = plan.alloc()
    plan.upload(f, c)
    plan.run_steps_inplace(c, 5)
    plan.normalize(c)
    plan.download(c, got)
    np.testing.assert_array_equal(got, want)


def test_pack_variant_on_a_nine_cell_row_in_place():
    """A pack variant on a row of 9 cells (two packs + one cell): served by the
    pack kernels, two blocks and in place (see
    test_pack_kernels_on_rows_no_pack_divides, test_inplace_pack_kernels_on_ragged_rows)."""
    grid, wall_u, inlet_u = geometries3d()["cavity"]  # nx = 9
    f = random_block(np.random.default_rng(3), grid.size, np.float32)
    want = make_oracle(grid, 1.0, wall_u).run(f.copy(), f.copy(), 4)
    plan = make_plan(grid, Precision.SINGLE, 1.0, wall_u)
    plan.set_variant(1008)
    c = plan.alloc()
    plan.upload(f, c)
    plan.run_steps_inplace(c, 4)
    plan.normalize(c)
    got = np.empty_like(f)
    plan.download(c, got)
    np.testing.assert_array_equal(got, want)


def test_never_writes_non_fluid_cells(rng):
    # test_kernels.py:205-219
    grid, wall_u, inlet_u = geometries3d()["channel"]
    f = random_block(rng, grid.size, np.float64)
    post = np.full_like(f, -7.5)
    make_plan(grid, Precision.DOUBLE, 1.3, wall_u, inlet_u).step(f, post)
    non_fluid = B.flatten_mask(grid) != B.FLUID
    assert (post[:, non_fluid] == -7.5).all()
    assert not (post[:, ~non_fluid] == -7.5).any()


def test_pure_streaming_at_omega_zero(rng):
    # omega = 0 turns the step into the pull permutation (test_kernels.py:152-164)
    from paper_2409_16781_b200.lattice import C
    nx, ny, nz = 6, 5, 7
    grid = B.open_mask(nx, ny, nz)
    f = random_block(rng, grid.size, np.float64)
    got = f.copy()
    make_plan(grid, Precision.DOUBLE, 0.0, (0, 0, 0)).step(f, got)
    fx, gx = to_xyzq(f, nx, ny, nz), to_xyzq(got, nx, ny, nz)
    for i in range(19):
        want = np.roll(fx[..., i], tuple(C[i]), axis=(0, 1, 2))
        np.testing.assert_array_equal(gx[..., i], want)


def test_flags_byte_identical(rng):
    for geom, (grid, wall_u, inlet_u) in geometries3d().items():
        plan = make_plan(grid, Precision.SINGLE, 1.0, wall_u, inlet_u)
        np.testing.assert_array_equal(plan.device_flags(), B.flatten_mask(grid))


@pytest.mark.parametrize("tag", ["f64", "f32", "f16"])
def test_macro_bitwise_and_diagnostics(tag, rng):
    grid, wall_u, inlet_u = geometries3d()["channel"]
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    f = random_block(rng, grid.size, prec.storage)
    orc = make_oracle(grid, 1.0, wall_u, inlet_u)
    plan = make_plan(grid, prec, 1.0, wall_u, inlet_u)
    d = plan.alloc()
    plan.upload(f, d)
    got = [t.cpu().numpy().transpose(2, 1, 0) for t in plan.macro(d)]
    for g, w in zip(got, orc.macro(f)):
        np.testing.assert_array_equal(g, w)
    gd, wd = plan.diagnostics(d), orc.diagnostics(f)
    for key in wd:
        assert gd[key] == pytest.approx(wd[key], rel=1e-12, abs=1e-12), key
    assert gd["fluid_cells"] == np.count_nonzero(grid == 0)
    f[3, 17] = np.nan
    f[11, 5] = np.inf  # (both representable in every storage dtype)
    plan.upload(f, d)
    assert plan.diagnostics(d)["nonfinite"] == 2


@pytest.mark.parametrize("geom", ["channel40", "channel"])  # pack kernel / one cell per thread
@pytest.mark.parametrize("tag", ["f64", "f32", "f16"])
def test_nonfinite_count_is_exact(tag, geom, rng):
    """The diagnostics count non-finite VALUES (the oracle's definition), and the
    kernels look at the individual values only where a cell's sum is non-finite:
    several per cell, +inf and -inf in one cell (their sum is a NaN), wall cells,
    and - in float64 - finite terms whose sum overflows (not a non-finite value)."""
    grid, wall_u, inlet_u = geometries3d()[geom]
    prec = PREC[tag]
    f = random_block(rng, grid.size, prec.storage)
    plan = make_plan(grid, prec, 1.0, wall_u, inlet_u)
    d = plan.alloc()
    if tag == "f64":
        big = f.copy()
        big[:, 7] = 1.7e308  # 19 finite terms, an infinite sum
        big[2, 9] = -1.7e308
        plan.upload(big, d)
        assert plan.diagnostics(d)["nonfinite"] == 0
    cells = rng.choice(grid.size, size=40, replace=False)
    for n, c in enumerate(cells):
        qs = rng.choice(19, size=1 + n % 5, replace=False)
        f[qs, c] = rng.choice([np.nan, np.inf, -np.inf], size=len(qs))
    f[[1, 3], cells[0]] = [np.inf, -np.inf]
    f[:, cells[1]] = np.nan
    want = int(np.count_nonzero(~np.isfinite(f)))
    assert want > 40
    plan.upload(f, d)
    assert plan.diagnostics(d)["nonfinite"] == want
    assert make_oracle(grid, 1.0, wall_u, inlet_u, prec).diagnostics(f)["nonfinite"] == want


def test_ldc64_fp64_100_steps_bitwise():
    """BASELINE.json config 1: D3Q19 BGK lid-driven cavity 64^3, 100 steps,
    fp64, through the reference-shaped API (cases.init + engine.run)."""
    from paper_2409_16781_b200 import cases, engine
    spec = cases.CaseSpec("ldc", 64, 64, 64, re=100.0, u0=0.1)
    state = cases.init(spec, Precision.DOUBLE)
    f0 = state.f_pre.data.copy()
    stats = engine.run(state, engine.RunConfig(steps=100, precision=Precision.DOUBLE))
    assert state.t == 100 and stats.mlups > 0
    orc = CpuOracle(64, 64, 64, state.mask, state.params.omega, state.wall_u,
                    threads=8)
    want = orc.run(f0.copy(), f0.copy(), 100)
    np.testing.assert_array_equal(state.f_pre.data, want)
    rho, ux, uy, uz = state.macro()
    for g, w in zip((rho, ux, uy, uz), orc.macro(want)):
        np.testing.assert_array_equal(g, w)
    assert ux.max() > 1e-3  # the lid drags the fluid along +x


@pytest.mark.parametrize("case,tag,tol", [("ldc24", "f64", 1e-13), ("tgv16", "f64", 1e-13),
                                          ("vks48", "f64", 1e-13), ("ldc24", "f32", 1e-5)])
def test_z_projection_bridge_to_lb2d(case, tag, tol, golden):
    """The CUDA path against the REAL reference: a z-invariant, z-periodic
    D3Q19 run summed over c_z equals the lb2d D2Q9 run (golden vectors from
    tests/golden/make_golden.py)."""
    p = f"{case}_{tag}_"
    nx, ny, steps = int(golden[p + "nx"]), int(golden[p + "ny"]), int(golden[p + "steps"])
    nz = 4
    prec = PREC[tag]
    from paper_2409_16781_b200.kernels import KernelPlan
    wu = golden[p + "wall_u"]
    plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, extrude_mask(golden[p + "mask"], nx, ny, nz),
                      float(golden[p + "omega"]), (wu[0], wu[1], 0.0),
                      inlet_u=float(golden[p + "inlet_u"]))
    f0 = lift_2d(golden[p + "f0"], nz)
    da, db = plan.alloc(), plan.alloc()
    plan.upload(f0, da)
    plan.upload(f0, db)
    newest, _, _ = plan.run_steps(da, db, steps)
    got = np.empty_like(f0)
    plan.download(newest, got)
    want = golden[p + "f"].astype(np.float64)
    proj = project_2d(got, nz)
    scale = np.abs(want).max()
    assert np.abs(proj - want[None]).max() / scale <= tol


@pytest.mark.parametrize("tag", ["f64", "f32", "f16"])
def test_engine_run_on_chained_outlets_falls_back_to_strict_stores(tag, rng):
    """engine.run must stay bit-exact on a geometry where pass-through is
    invalid (chained outlet cells) by keeping the strict store mode."""
    from paper_2409_16781_b200 import engine
    from paper_2409_16781_b200.lattice import RelaxationParams
    grid, wall_u, inlet_u = geometries3d()["open_chain"]
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    rho = rng.uniform(0.9, 1.1, size=grid.shape)
    u = rng.uniform(-0.05, 0.05, size=(3,) + grid.shape)
    state = engine.state_from_macroscopic(rho, u[0], u[1], u[2], grid, Layout.ROW, prec,
                                          params=RelaxationParams.from_omega(1.2),
                                          inlet_u=inlet_u)
    f0 = state.f_pre.data.copy()
    engine.run(state, engine.RunConfig(steps=9, precision=prec))
    want = make_oracle(grid, 1.2, wall_u, inlet_u).run(f0.copy(), f0.copy(), 9)
    np.testing.assert_array_equal(state.f_pre.data, want)


@pytest.mark.parametrize("tag", ["f32", "f64", "f16"])
def test_graph_replay_never_changes_bits(tag):
    """mlb_run_steps / mlb_run_steps_inplace replay runs of steps from a CUDA
    graph on small domains (mlb_plan_set_graph): the very launches of the plain
    loop, so the same bits - for run lengths around the 32-step graph unit, odd
    and even, two blocks and in place, with walls and open boundaries."""
    from paper_2409_16781_b200.kernels import KernelPlan
    prec = {"f64": Precision.DOUBLE, "f32": Precision.SINGLE, "f16": Precision.MIXED1}[tag]
    for geom in ("cavity16", "channel40"):
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        flags = B.flatten_mask(grid)
        f = random_block(np.random.default_rng(20240917), grid.size, prec.storage)
        want = {}
        for steps in (9, 32, 71):
            for graph in (0, 1):
                plan = KernelPlan(nx, ny, nz, Layout.ROW, prec, flags, 1.3, wall_u, inlet_u=inlet_u)
                plan.set_graph(graph)
                a, b = plan.alloc(), plan.alloc()
                plan.upload(f, a)
                plan.upload(f, b)
                newest, _, _ = plan.run_steps(a, b, steps)
                got = np.empty_like(f)
                plan.download(newest, got)
                if graph == 0:
                    want[steps] = got
                else:
                    np.testing.assert_array_equal(got, want[steps])
                    # a second call reuses the cached graph (same blocks, same plan state)
                    newest2, _, _ = plan.run_steps(newest, b if newest is a else a, steps)
                    # and in place, from both representations
                    c = plan.alloc()
                    plan.upload(f, c)
                    plan.set_variant(1008 if tag != "f16" else 2008)
                    plan.run_steps_inplace(c, 1)            # now shifted: the replay starts from repr 1
                    plan.run_steps_inplace(c, steps - 1)
                    plan.normalize(c)
                    got = np.empty_like(f)
                    plan.download(c, got)
                    np.testing.assert_array_equal(got, want[steps])
                plan.close()
    orc = CpuOracle(nx, ny, nz, flags, 1.3, wall_u, inlet_u)
    np.testing.assert_array_equal(orc.run(f.copy(), f.copy(), 71), want[71])


def _stage_geometries():
    """Walls inside and between packs, ragged rows (100, 250) that span one or
    several warp columns, inlet / outlet faces, and a fully periodic box where
    the x wrap is live."""
    prng = np.random.default_rng(11)
    cav = B.cavity_mask(100, 16, 6)
    cav[40:47, 5:9, 2:4] = B.SOLID
    cav[77, 11, 3] = B.MOVING_WALL
    chan = B.channel_mask(128, 16, 6, B.sphere_cells(128, 16, 6, 6, 30.0, 8.0, 2.5))
    per = B.open_mask(250, 8, 5)
    u = prng.random(per.shape)
    per[u < 0.04] = B.SOLID
    per[u > 0.98] = B.MOVING_WALL
    return {"cavity100": (cav, (0.05, 0.0, -0.03), 0.0),
            "channel128": (chan, (0.0, 0.0, 0.0), 0.06),
            "periodic250": (per, (0.02, 0.03, -0.04), 0.0)}


@pytest.mark.parametrize("mode", ["strict", "passthrough", "slab"])
@pytest.mark.parametrize("tag", ["f16", "m2", "f32", "f64"])
@pytest.mark.parametrize("geom", ["cavity100", "channel128", "periodic250"])
def test_staged_kernel_never_changes_bits(geom, tag, mode, rng):
    """step_stage_kernel (variant 4000): the row segments a warp pulls from are
    staged in shared memory by cp.async one row ahead of the arithmetic.  What
    follows the loads is the direct kernel's code, so - like tiling in the
    reference (test_kernels.py:107-126) - it never changes a bit: strict and
    pass-through stores, fused open-boundary pass, ragged rows, periodic wrap
    in x / y / z, and z-slabs with halo planes (plane ranges, boundary first)."""
    from paper_2409_16781_b200 import slab
    grid, wall_u, inlet_u = _stage_geometries()[geom]
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    f = random_block(rng, grid.size, prec.storage)
    sentinel = random_block(rng, grid.size, prec.storage)
    if mode != "strict":
        sentinel = f.copy()
    omega, steps = 1.55, 4
    want = make_oracle(grid, omega, wall_u, inlet_u, prec).run(f.copy(), sentinel.copy(), steps)
    if mode == "slab":
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        lo, hi = slab.slab_halo_flags(flags, nx, ny, 0, nz)
        plan = make_plan(grid, prec, omega, wall_u, inlet_u, halo_lo=lo, halo_hi=hi, slab=True)
    else:
        plan = make_plan(grid, prec, omega, wall_u, inlet_u)
    plan.set_variant(4000)
    if tag in ("f16", "m2"):
        assert "step_stage_kernel" in plan.kernel_name
    else:   # fp32 / fp64 sit at the HBM roofline with the direct kernel: the variant falls back
        assert "stage" not in plan.kernel_name
    plan.set_passthrough(mode != "strict")
    a, b = plan.alloc(), plan.alloc()
    a.tensor.fill_(float("nan"))
    b.tensor.fill_(float("nan"))
    plan.upload(f, a)
    plan.upload(sentinel, b)
    if mode == "slab":
        runner = slab.DistSlab(slab.CudaStepper(plan), nz)
        runner.exchange(a)
        newest, _ = runner.run(a, b, steps)
    else:
        newest, _, _ = plan.run_steps(a, b, steps)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("passthrough", [False, True])
@pytest.mark.parametrize("tag,variant", [("f32", 1008), ("f32", 1016), ("f32", 2032), ("f16", 2008),
                                         ("f16", 3016), ("m2", 2016), ("f64", 1008)])
@pytest.mark.parametrize("shape", [(13, 6, 5), (15, 5, 4), (101, 4, 3), (131, 9, 3)])
def test_pack_kernels_on_rows_no_pack_divides(shape, tag, variant, passthrough, rng):
    """Rows whose length the pack does not divide end in a pack of real cells +
    row padding; the cell at x = nx-1 then sits inside a pack and its x+1
    neighbour is cell 0 of the row (periodic wrap), not the padding.  Periodic
    box with scattered walls (the wrap is live) and a closed cavity."""
    nx, ny, nz = shape
    prec = PREC[tag]
    for kind in ("periodic", "cavity"):
        grid = B.open_mask(nx, ny, nz) if kind == "periodic" else B.cavity_mask(nx, ny, nz)
        u = np.random.default_rng(nx).random(grid.shape)
        grid[(u < 0.05) & (grid == B.FLUID)] = B.SOLID
        grid[(u > 0.97) & (grid == B.FLUID)] = B.MOVING_WALL
        f = random_block(rng, grid.size, prec.storage)
        sentinel = f.copy() if passthrough else random_block(rng, grid.size, prec.storage)
        wall_u = (0.04, -0.02, 0.03)
        want = make_oracle(grid, 1.7, wall_u, 0.0, prec).run(f.copy(), sentinel.copy(), 3)
        plan = make_plan(grid, prec, 1.7, wall_u)
        plan.set_variant(variant)
        plan.set_passthrough(passthrough)
        a, b = plan.alloc(), plan.alloc()
        plan.upload(f, a)
        plan.upload(sentinel, b)
        newest, _, _ = plan.run_steps(a, b, 3)
        got = np.empty_like(f)
        plan.download(newest, got)
        np.testing.assert_array_equal(got, want)
