"""Seeded random geometries through every kernel family, against the oracle,
bit for bit.  Each case draws its own grid shape (ragged and pack-aligned row
lengths), flag field (solid and moving grains, inlet / outlet cells wherever
the reference would accept them), relaxation rate, wall and inlet velocity,
storage mode, kernel variant and step count; then runs
  * the two-buffer kernels, strict stores with arbitrary never-written cells,
  * the two-buffer kernels with pass-through stores (when the library accepts
    the geometry),
  * the in-place kernels (when the library accepts the geometry),
  * the z-slab driver with the fused peer-store exchange (ring closed on the
    slab itself), two blocks and - where accepted - one block,
and requires the oracle's bits every time."""

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.fields import Layout, Precision

from .helpers import random_block

pytestmark = pytest.mark.gpu

PREC = {"f32": Precision.SINGLE, "f64": Precision.DOUBLE, "f16": Precision.MIXED1,
        "m2": Precision.MIXED2}
SCALAR = [32, 64, 128, 256]
PACKS = {"f32": [1008, 1016, 1032, 2008, 2016, 2032], "f64": [1008, 1016, 1032],
         "f16": [2008, 2016, 2032, 3008, 3016, 3032, 4000], "m2": [2008, 2016, 2032, 4000]}


BIG = __import__("os").environ.get("MLB_FUZZ_SCALE") == "big"


def draw_case(seed):
    r = np.random.default_rng(seed)
    tag = ["f32", "f64", "f16", "m2"][r.integers(4)]
    aligned = r.random() < 0.7
    nx = int(r.integers(2, 19)) * 4 if aligned else int(r.integers(5, 40))
    ny, nz = int(r.integers(3, 9)), int(r.integers(3, 8))
    if BIG:   # MLB_FUZZ_SCALE=big: grids on which concurrent launches really overlap
        nx = int(r.integers(16, 41)) * 4 if aligned else int(r.integers(60, 170))
        ny, nz = int(r.integers(8, 40)), int(r.integers(6, 24))
    grid = B.open_mask(nx, ny, nz)
    u = r.random(grid.shape)
    p_solid, p_move = r.choice([0.0, 0.05, 0.25]), r.choice([0.0, 0.03, 0.1])
    grid[u < p_solid] = B.SOLID
    grid[u > 1.0 - p_move] = B.MOVING_WALL
    if r.random() < 0.4:          # a closed box around it
        grid[0], grid[-1] = B.SOLID, B.SOLID
        grid[:, 0], grid[:, -1] = B.SOLID, B.MOVING_WALL
    inlet_u = 0.0
    if r.random() < 0.5:          # open-boundary cells: anywhere, as index lists allow
        inlet_u = float(r.uniform(0.01, 0.08))
        for _ in range(int(r.integers(1, 4))):
            x = int(r.integers(0, nx))
            grid[x, r.integers(0, ny), :] = B.INLET
        for _ in range(int(r.integers(1, 4))):
            x = int(r.integers(1, nx))      # an outlet cell at x = 0 is rejected by design
            grid[x, :, r.integers(0, nz)] = B.OUTLET
    omega = float(r.choice([0.0, r.uniform(0.2, 1.99)], p=[0.05, 0.95]))
    wall_u = tuple(float(v) for v in r.uniform(-0.06, 0.06, 3))
    # (pack kernels on ragged rows too: the last pack of a row is real cells + padding)
    variant = int(r.choice(PACKS[tag] if r.random() < 0.75 else SCALAR))
    steps = int(r.integers(1, 5)) if r.random() < 0.85 else int(r.integers(8, 13))
    return tag, grid, omega, wall_u, inlet_u, variant, steps


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("MLB_FUZZ_CASES", "120"))))
def test_random_case_every_kernel_family_bitwise(seed):
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    tag, grid, omega, wall_u, inlet_u, variant, steps = draw_case(seed)
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    mask = B.flatten_mask(grid)
    rng = np.random.default_rng(1000 + seed)
    f = random_block(rng, grid.size, prec.storage)
    sentinel = random_block(rng, grid.size, prec.storage)
    orc = CpuOracle(nx, ny, nz, mask, omega, wall_u, inlet_u,
                    compute=np.float64 if prec is Precision.MIXED2 else None)

    def plan_for(**kw):
        p = KernelPlan(nx, ny, nz, Layout.ROW, prec, mask, omega, wall_u, inlet_u=inlet_u, **kw)
        p.set_variant(variant)
        p.set_inplace_layout(seed % 3 == 0)      # thread layout of the in-place pull half
        p.set_graph(seed % 2)                    # CUDA-graph replay of the loop (runs of >= 8 steps)
        return p

    # two buffers, strict: arbitrary never-written cells in the second buffer
    want = orc.run(f.copy(), sentinel.copy(), steps)
    plan = plan_for()
    a, b = plan.alloc(), plan.alloc()
    plan.upload(f, a)
    plan.upload(sentinel, b)
    newest, _, _ = plan.run_steps(a, b, steps)
    got = np.empty_like(f)
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want, err_msg=f"strict, case {seed}")
    np.testing.assert_array_equal(plan.device_flags(), mask)

    # from here on both buffers start identical (engine.py:148)
    want = orc.run(f.copy(), f.copy(), steps)
    try:
        plan.set_passthrough(True)
        fused = True
    except ValueError:
        fused = False             # chained outlet cells: refused by design
    if fused:
        plan.upload(f, a)
        plan.upload(f, b)
        newest, _, _ = plan.run_steps(a, b, steps)
        plan.download(newest, got)
        np.testing.assert_array_equal(got, want, err_msg=f"pass-through, case {seed}")

    # in place, when the library serves this geometry with this variant
    plan.upload(f, a)
    a.repr = 0
    try:
        plan.run_steps_inplace(a, steps)
        inplace = True
    except ValueError:
        inplace = False
    if inplace:
        plan.normalize(a)
        plan.download(a, got)
        np.testing.assert_array_equal(got, want, err_msg=f"in place, case {seed}")
    plan.close()

    # the whole run on host blocks with upload, steps and download overlapped chunk by
    # chunk (mlb_run_steps_host, one plane per chunk): needs a domain closed in z, so the
    # same case with planes 0 and nz-1 walled off
    if nz >= 4:
        gz = grid.copy()
        gz[:, :, 0] = B.SOLID
        gz[:, :, -1] = B.MOVING_WALL
        mz = B.flatten_mask(gz)
        oz = CpuOracle(nx, ny, nz, mz, omega, wall_u, inlet_u,
                       compute=np.float64 if prec is Precision.MIXED2 else None)
        wz = oz.run(f.copy(), f.copy(), steps)
        pz = KernelPlan(nx, ny, nz, Layout.ROW, prec, mz, omega, wall_u, inlet_u=inlet_u,
                        defer_flags=bool(seed % 2))
        pz.set_variant(variant)
        a, b = pz.alloc(), pz.alloc()
        out = np.empty_like(f)
        _, _, _, overlapped = pz.run_host(f, out, a, b, steps, chunk_planes=1)
        assert overlapped
        np.testing.assert_array_equal(out, wz, err_msg=f"overlapped host run, case {seed}")
        pz.close()

    # the z-slab driver, ring closed on the slab itself
    flags3 = mask.reshape(nz, ny, nx)
    lo, hi = slab.slab_halo_flags(flags3, nx, ny, 0, nz)
    plan = plan_for(halo_lo=lo, halo_hi=hi, slab=True)
    if fused:
        plan.set_passthrough(True)
    a, b = plan.alloc(), plan.alloc()
    for blk in (a, b):
        blk.tensor.fill_(float("nan"))
        plan.upload(f, blk)
    ring = slab.PeerRing(plan, [a, b])
    runner = slab.DistSlab(slab.CudaStepper(plan), nz, overlap=bool(seed % 2), ring=ring)
    runner.exchange(a)
    newest, _ = runner.run(a, b, steps)
    runner.finish()
    plan.download(newest, got)
    np.testing.assert_array_equal(got, want, err_msg=f"slab ring, case {seed}")
    ring.close()
    if inplace and 1000 <= variant < 4000:
        c = plan.alloc()
        c.tensor.fill_(float("nan"))
        plan.upload(f, c)
        ring = slab.PeerRing(plan, [c])
        runner = slab.DistSlab(slab.CudaStepper(plan), nz, overlap=bool(seed % 2), ring=ring)
        runner.exchange(c)
        runner.run_inplace(c, steps)
        runner.normalize(c)
        plan.download(c, got)
        np.testing.assert_array_equal(got, want, err_msg=f"in-place slab, case {seed}")
        ring.close()
    plan.close()


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("MLB_ENGINE_FUZZ_CASES", "40"))))
def test_random_engine_sequences_bitwise(seed):
    """The host layer on random cases: a random sequence of engine.run calls
    (two blocks / in place, with and without the overlapped host path, with output
    hooks), resident sessions advanced directly, host edits between runs, probed
    runs, diagnostics calls and a checkpoint round trip in the middle - the final
    populations must be the oracle's after the same sequence (the oracle carries
    both of its buffers along, as the reference's SimState does)."""
    import os
    import tempfile
    from paper_2409_16781_b200 import engine
    from paper_2409_16781_b200.fields import PopulationField
    from paper_2409_16781_b200.lattice import RelaxationParams
    tag, grid, omega, wall_u, inlet_u, variant, steps = draw_case(7000 + seed)
    if omega == 0.0:
        omega = 0.7          # RelaxationParams wants omega in (0, 2)
    prec = PREC[tag]
    nx, ny, nz = grid.shape
    mask = B.flatten_mask(grid)
    r = np.random.default_rng(9000 + seed)
    f = random_block(r, grid.size, prec.storage)
    orc = CpuOracle(nx, ny, nz, mask, omega, wall_u, inlet_u,
                    compute=np.float64 if prec is Precision.MIXED2 else None)

    def make_state(data, t=0):
        return engine.SimState(f_pre=PopulationField(data.copy(), nx, ny, nz, Layout.ROW),
                               f_post_=None, mask=mask, nx=nx, ny=ny, nz=nz, layout=Layout.ROW,
                               precision=prec, t=t, params=RelaxationParams.from_omega(omega),
                               wall_u=wall_u, inlet_u=inlet_u)

    # the oracle's two buffers travel with the sequence: a geometry that chains outlet
    # cells reads stale values of the second one (engine.py:179-180 of the reference)
    ora = {"pre": f.copy(), "post": f.copy()}

    def oracle_steps(n):
        newest = orc.run(ora["pre"], ora["post"], n)
        if newest is not ora["pre"]:
            ora["pre"], ora["post"] = ora["post"], ora["pre"]

    state, total = make_state(f), 0
    for _ in range(int(r.integers(2, 6))):
        k = int(r.integers(1, 10))
        op = int(r.integers(0, 9))
        inplace = bool(r.integers(0, 2))
        try:
            if op == 5:      # a host edit between runs (fluid cells: the reference's f_pre only)
                fluid = np.flatnonzero(mask == B.FLUID)
                if fluid.size:
                    cells = r.choice(fluid, size=min(5, fluid.size), replace=False)
                    q = int(r.integers(0, 19))
                    vals = random_block(r, cells.size, prec.storage)[q]
                    state.f_pre.data[q, cells] = vals
                    ora["pre"][q, cells] = vals
                k = 0
            elif op == 6:    # diagnostics of a host state: a temporary session, nothing changes
                rho, ux, uy, uz = state.macro()
                want_rho = ora["pre"].astype(np.float64).sum(axis=0).reshape(nz, ny, nx)
                np.testing.assert_allclose(rho.transpose(2, 1, 0), want_rho, rtol=1e-6)
                d = state.diagnostics()
                assert d["fluid_cells"] == int(np.count_nonzero(mask == B.FLUID))
                k = 0
            elif op == 7:    # a probed run: one step per launch, a device-side series
                fluid = np.flatnonzero(mask == B.FLUID)
                cell = int(fluid[0]) if fluid.size else 0
                pz, py, px = np.unravel_index(cell, (nz, ny, nx))
                stats = engine.run(state, engine.RunConfig(steps=k, precision=prec,
                                                           inplace=inplace),
                                   probe=(int(px), int(py), int(pz)))
                assert stats.probe_samples.shape == (k, 4)
            elif op == 8:    # the host asks for its second buffer (materialised on first use)
                assert state.f_post.data.shape == state.f_pre.data.shape
                k = 0
            if op >= 5:
                pass
            elif op == 0:    # plain run, maybe through the overlapped host path
                engine.run(state, engine.RunConfig(steps=k, precision=prec, inplace=inplace,
                                                   overlap_io=[None, False][int(r.integers(0, 2))]))
            elif op == 1:    # run with an output hook (finite check + host sync at cadence)
                seen = []
                engine.run(state, engine.RunConfig(steps=k, precision=prec, inplace=inplace,
                                                   output_every=2),
                           on_output=lambda st: seen.append(st.t))
                assert seen == [t for t in range(total + 1, total + k + 1) if t % 2 == 0]
            elif op == 2:    # resident session advanced directly, then a run on top of it
                sess = engine.open_session(state, engine.RunConfig(steps=1, precision=prec,
                                                                   inplace=inplace))
                sess.advance(k)
                total += k
                oracle_steps(k)
                k = int(r.integers(1, 6))
                engine.run(state, engine.RunConfig(steps=k, precision=prec, inplace=inplace))
                sess.close()
            elif op == 3:    # checkpoint round trip, then carry on from the restored state
                with tempfile.TemporaryDirectory() as d:
                    path = os.path.join(d, "c.mlb")
                    engine.checkpoint(state, path)
                    back = engine.restore(path)
                assert back.t == state.t
                # (the file holds the first buffer only; restore starts both identical,
                # engine.py:329 of the reference)
                ora["post"] = ora["pre"].copy()
                state = make_state(back.f_pre.data, back.t)
                engine.run(state, engine.RunConfig(steps=k, precision=prec, inplace=inplace))
            else:            # the one-step convenience call, k times
                for _ in range(k):
                    engine.step(state)
        except ValueError as exc:
            # geometries the in-place update cannot serve are refused BEFORE any step
            assert inplace and "in-place" in str(exc), exc
            if state.session is not None:
                state.session.close()
            continue
        except engine.DivergenceError:
            # random populations may blow up: the finite check at output cadence then
            # raises at the step the ORACLE's populations turn non-finite too, with the
            # diverged populations in the host arrays (engine.py:258-259 of the reference)
            assert op == 1
            oracle_steps(state.t - total)
            assert not np.isfinite(ora["pre"].astype(np.float64)).all()
            total = state.t
            break
        total += k
        oracle_steps(k)
        assert state.t == total
        if k and state.f_post_ is not None:
            # after a two-block run the buffer swapped out last is the previous step's
            # state in the reference too; an in-place run has no second block (copy)
            ran_inplace = inplace and op in (0, 1, 2, 7)
            want_post = ora["pre"] if ran_inplace else ora["post"]
            np.testing.assert_array_equal(state.f_post_.data, want_post,
                                          err_msg=f"second buffer, case {seed}, op {op}")
    want = ora["pre"]
    if state.session is not None:
        state.session.close()
    np.testing.assert_array_equal(state.f_pre.data, want, err_msg=f"engine sequence, case {seed}")
