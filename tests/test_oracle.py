"""Pin the CPU oracle (oracle/d3q19_oracle.c) before trusting it:

1. against the REAL reference through the z-projection bridge - golden
   vectors produced by lb2d itself (tests/golden/make_golden.py);
2. against the reference's known answers and invariants (omega = 0 is a
   roll, conservation, never-written cells, inlet/outlet semantics);
3. against an independent explicit-loop numpy oracle (oracle/ref3d.py) on
   genuinely 3-D geometries;
4. partition invariance: any number of z-slabs, any thread count, same bits.
"""

import numpy as np
import pytest

from oracle import cpu
from oracle.cpu import CpuOracle, SlabOracle
from oracle.ref3d import kahan_sum, ref3d_open_pass, ref3d_step
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import lattice as L
from paper_2409_16781_b200.slab import partition

from .helpers import (extrude_mask, from_xyzq, geometries3d, lift_2d, project_2d,
                      random_block, to_xyzq)


def oracle_for(grid, omega, wall_u, inlet_u=0.0, threads=2):
    nx, ny, nz = grid.shape
    return CpuOracle(nx, ny, nz, B.flatten_mask(grid), omega, wall_u, inlet_u, threads)


# ---- 1. the bridge to the real reference -----------------------------------
class TestBridgeToLb2d:
    @pytest.mark.parametrize("case,tag,tol", [
        ("ldc24", "f64", 1e-13), ("tgv16", "f64", 1e-13), ("vks48", "f64", 1e-13),
        ("ldc24", "f32", 1e-5), ("ldc24", "m2", 1e-6)])
    @pytest.mark.parametrize("nz", [1, 4])
    def test_engine_runs(self, case, tag, tol, nz, golden):
        """LDC, TGV and channel+disk (inlet/outlet pass included) through
        lb2d's engine.run vs the D3Q19 oracle summed over c_z."""
        p = f"{case}_{tag}_"
        nx, ny, steps = (int(golden[p + k]) for k in ("nx", "ny", "steps"))
        wu = golden[p + "wall_u"]
        orc = CpuOracle(nx, ny, nz, extrude_mask(golden[p + "mask"], nx, ny, nz),
                        float(golden[p + "omega"]), (wu[0], wu[1], 0.0),
                        float(golden[p + "inlet_u"]), threads=4,
                        compute=np.float64 if tag == "m2" else None)
        f0 = lift_2d(golden[p + "f0"], nz)
        got = orc.run(f0.copy(), f0.copy(), steps)
        want = golden[p + "f"].astype(np.float64)
        err = np.abs(project_2d(got, nz) - want[None]).max() / np.abs(want).max()
        assert err <= tol
        # macroscopic fields: rho, ux, uy equal lb2d's, uz identically zero
        rho, ux, uy, uz = orc.macro(got)
        scale = max(np.abs(golden[p + "ux"]).max(), 1e-30)
        for z in range(nz):
            assert np.abs(rho[:, :, z] - golden[p + "rho"]).max() <= tol
            assert np.abs(ux[:, :, z] - golden[p + "ux"]).max() <= tol * max(1.0, 1 / scale) * scale + tol
            assert np.abs(uy[:, :, z] - golden[p + "uy"]).max() <= tol * max(1.0, 1 / scale) * scale + tol
        assert np.abs(uz).max() <= (1e-15 if tag == "f64" else 1e-7)
        if tag == "m2":
            # lb2d's mixed2 run (float planes, double arithmetic) is closer to its
            # double run than its single run is: the mode does what it says
            d64 = golden["ldc24_f64_f"]
            e_m2 = np.abs(golden["ldc24_m2_f"].astype(np.float64) - d64).max()
            e_f32 = np.abs(golden["ldc24_f32_f"].astype(np.float64) - d64).max()
            assert e_m2 < e_f32

    @pytest.mark.parametrize("geom", ["cavity", "channel", "periodic"])
    def test_one_step_on_reference_kernel_geometries(self, geom, golden):
        """One fused step on the reference's three kernel-test geometries
        (test_kernels.py:25-61), random populations, omega 1.41: vs lb2d's
        numba kernel AND vs lb2d's independent ref_step."""
        grid2 = golden[f"k1_{geom}_grid"]
        nx, ny = grid2.shape
        nz = 3
        wu = golden[f"k1_{geom}_wall_u"]
        flags = extrude_mask(np.ascontiguousarray(grid2.T).reshape(-1), nx, ny, nz)
        orc = CpuOracle(nx, ny, nz, flags, 1.41, (wu[0], wu[1], 0.0))
        f0 = lift_2d(golden[f"k1_{geom}_f0"], nz)
        post = f0.copy()
        orc.step(f0, post)
        proj = project_2d(post, nz)
        np.testing.assert_allclose(proj[1], golden[f"k1_{geom}_numba"], rtol=1e-13, atol=1e-15)
        want = golden[f"k1_{geom}_refstep"]  # (nx, ny, 9)
        got = proj[2].reshape(9, ny, nx).transpose(2, 1, 0)
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-15)


# ---- 2. known answers and invariants ----------------------------------------
class TestInvariants:
    def test_omega_zero_is_the_pull_permutation(self, rng):
        nx, ny, nz = 6, 5, 4
        grid = B.open_mask(nx, ny, nz)
        f = random_block(rng, grid.size, np.float64)
        got = f.copy()
        oracle_for(grid, 0.0, (0, 0, 0)).step(f, got)
        fx, gx = to_xyzq(f, nx, ny, nz), to_xyzq(got, nx, ny, nz)
        for i in range(19):
            np.testing.assert_array_equal(
                gx[..., i], np.roll(fx[..., i], tuple(L.C[i]), axis=(0, 1, 2)))

    def test_periodic_conservation(self, rng):
        grid = B.open_mask(8, 6, 5)
        f = random_block(rng, grid.size, np.float64)
        post = f.copy()
        oracle_for(grid, 1.91, (0, 0, 0)).step(f, post)
        assert kahan_sum(post) == pytest.approx(kahan_sum(f), rel=1e-14)
        for c in (L.CX, L.CY, L.CZ):
            assert kahan_sum(c[:, None] * post) == pytest.approx(
                kahan_sum(c[:, None] * f), rel=1e-12, abs=1e-12)

    def test_closed_box_conserves_mass(self):
        # acceptance c02 / test_engine.py:132-137 in 3-D: walls exchange momentum, not mass
        grid = B.cavity_mask(10, 9, 8)
        orc = oracle_for(grid, 1.2, (0.1, 0.0, 0.0))
        f = np.repeat(L.W[:, None], grid.size, axis=1).copy()
        m0 = kahan_sum(f)
        out = orc.run(f, f.copy(), 150)
        assert kahan_sum(out) == pytest.approx(m0, rel=1e-13)

    def test_never_writes_non_fluid_cells(self, rng):
        grid, wall_u, inlet_u = geometries3d()["channel"]
        f = random_block(rng, grid.size, np.float64)
        post = np.full_like(f, -7.5)
        oracle_for(grid, 1.3, wall_u, inlet_u).step(f, post)
        non_fluid = B.flatten_mask(grid) != B.FLUID
        assert (post[:, non_fluid] == -7.5).all()
        assert not (post[:, ~non_fluid] == -7.5).any()

    def test_moving_lid_drags_adjacent_fluid(self):
        grid = B.cavity_mask(12, 12, 6)
        orc = oracle_for(grid, 1.0, (0.1, 0.0, 0.0))
        f = np.repeat(L.W[:, None], grid.size, axis=1).copy()
        out = orc.run(f, f.copy(), 20)
        _, ux, _, _ = orc.macro(out)
        assert ux[1:-1, -2, 1:-1].mean() > 1e-3

    def test_inlet_outlet_semantics(self, rng):
        # test_engine.py:184-203: inlet <- equilibrium(1, u_in, 0), outlet <- fresh west neighbour
        grid, wall_u, inlet_u = geometries3d()["channel"]
        orc = oracle_for(grid, 1.1, wall_u, inlet_u)
        f = random_block(rng, grid.size, np.float64)
        post = f.copy()
        orc.step(f, post)
        before = post.copy()
        orc.open_pass(post)
        flat = B.flatten_mask(grid)
        eq = L.equilibrium(1.0, inlet_u, 0.0, 0.0)
        np.testing.assert_array_equal(post[:, flat == B.INLET],
                                      np.repeat(eq[:, None], (flat == B.INLET).sum(), 1))
        out_idx = np.nonzero(flat == B.OUTLET)[0]
        np.testing.assert_array_equal(post[:, out_idx], before[:, out_idx - 1])
        untouched = (flat != B.INLET) & (flat != B.OUTLET)
        np.testing.assert_array_equal(post[:, untouched], before[:, untouched])

    def test_inlet_values_in_compute_dtype(self):
        for dt in (np.float32, np.float64):
            np.testing.assert_array_equal(cpu.equilibrium(1.0, 0.07, 0.0, 0.0, dt),
                                          L.equilibrium(1.0, 0.07, 0.0, 0.0, dtype=dt))

    def test_outlet_at_x0_rejected(self):
        grid = B.open_mask(4, 4, 2)
        grid[0, 1, 0] = B.OUTLET
        orc = oracle_for(grid, 1.0, (0, 0, 0))
        f = np.ones((19, grid.size))
        with pytest.raises(RuntimeError):
            orc.open_pass(f)

    def test_diagnostics_against_numpy(self, rng):
        grid, wall_u, inlet_u = geometries3d()["cavity"]
        orc = oracle_for(grid, 1.0, wall_u)
        f = random_block(rng, grid.size, np.float64)
        d = orc.diagnostics(f)
        fluid = B.flatten_mask(grid) == 0
        rho = f.sum(0)
        m = np.stack([(c[:, None] * f).sum(0) for c in (L.CX, L.CY, L.CZ)])
        assert d["mass"] == pytest.approx(kahan_sum(f), rel=1e-13)
        assert d["fluid_cells"] == fluid.sum() and d["nonfinite"] == 0
        assert d["px"] == pytest.approx(m[0][fluid].sum(), rel=1e-12)
        ke = 0.5 * ((m ** 2).sum(0) / rho)[fluid].sum()
        assert d["kinetic_energy"] == pytest.approx(ke, rel=1e-12)
        assert d["max_u"] == pytest.approx((np.sqrt((m ** 2).sum(0)) / rho)[fluid].max(), rel=1e-13)


class TestMixed1Storage:
    @pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel40", "periodic8"])
    def test_half_storage_is_the_float_kernel_between_two_casts(self, geom, rng):
        """The reference defines MIXED1 through float32 bridge planes
        (kernels.py:447-455): f16 -> f32 is exact, the float kernel runs,
        f32 -> f16 rounds to nearest.  The half-storage oracle must equal
        exactly that, step after step, never-written cells included."""
        grid, wall_u, inlet_u = geometries3d()[geom]
        orc = oracle_for(grid, 1.3, wall_u, inlet_u)
        f16 = random_block(rng, grid.size, np.float16)
        a, b = f16.copy(), random_block(rng, grid.size, np.float16)
        a32, b32 = a.astype(np.float32), b.astype(np.float32)
        for _ in range(4):
            orc.step(a, b)
            orc.open_pass(b)
            orc.step(a32, b32)
            orc.open_pass(b32)
            b32 = b32.astype(np.float16).astype(np.float32)  # the bridge's store + reload
            np.testing.assert_array_equal(b, b32.astype(np.float16))
            a, b, a32, b32 = b, a, b32, a32

    def test_macro_upcasts_exactly(self, rng):
        grid, wall_u, inlet_u = geometries3d()["periodic8"]
        orc = oracle_for(grid, 1.0, wall_u)
        f16 = random_block(rng, grid.size, np.float16)
        for got, want in zip(orc.macro(f16), orc.macro(f16.astype(np.float64))):
            np.testing.assert_array_equal(got, want)


class TestMixed2Storage:
    @pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel40", "periodic8"])
    def test_float_storage_is_the_double_kernel_between_two_casts(self, geom, rng):
        """The reference's MIXED2 (fields.py:25): its kernel, compiled for
        float64, upcasts every load (`one * fpre[...]`, kernels.py:80-96) and the
        store into the float32 plane rounds to nearest.  The oracle's
        float-storage / double-compute instantiation must equal the double
        kernel between an exact upcast and one rounding, step after step,
        never-written cells included."""
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        mask = B.flatten_mask(grid)
        m2 = CpuOracle(nx, ny, nz, mask, 1.3, wall_u, inlet_u, compute=np.float64)
        dbl = CpuOracle(nx, ny, nz, mask, 1.3, wall_u, inlet_u)
        a, b = random_block(rng, grid.size, np.float32), random_block(rng, grid.size, np.float32)
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        for _ in range(4):
            m2.step(a, b)
            m2.open_pass(b)
            dbl.step(a64, b64)
            dbl.open_pass(b64)
            b64 = b64.astype(np.float32).astype(np.float64)   # the store's rounding + the next load
            np.testing.assert_array_equal(b, b64.astype(np.float32))
            a, b, a64, b64 = b, a, b64, a64
        # and it is NOT the float kernel
        s = CpuOracle(nx, ny, nz, mask, 1.3, wall_u, inlet_u)
        x = random_block(rng, grid.size, np.float32)
        y1, y2 = x.copy(), x.copy()
        s.step(x, y1)
        m2.step(x, y2)
        assert not np.array_equal(y1, y2)


# ---- 3. the independent naive oracle on 3-D geometries ----------------------
class TestAgainstNaiveOracle:
    @pytest.mark.parametrize("geom", list(geometries3d()))
    def test_one_step(self, geom, rng):
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        f = random_block(rng, grid.size, np.float64)
        got = f.copy()
        oracle_for(grid, 1.41, wall_u, inlet_u).step(f, got)
        want = ref3d_step(to_xyzq(f, nx, ny, nz), grid, 1.41, wall_u)
        np.testing.assert_allclose(to_xyzq(got, nx, ny, nz), want, rtol=1e-12, atol=1e-15)

    def test_five_steps_with_open_pass(self, rng):
        # test_kernels.py:63-79 tolerance
        grid, wall_u, inlet_u = geometries3d()["channel"]
        nx, ny, nz = grid.shape
        f = random_block(rng, grid.size, np.float64)
        got = oracle_for(grid, 0.9, wall_u, inlet_u).run(f.copy(), f.copy(), 5)
        fx = to_xyzq(f, nx, ny, nz)
        for _ in range(5):
            fx = ref3d_open_pass(ref3d_step(fx, grid, 0.9, wall_u), grid, inlet_u)
        np.testing.assert_allclose(to_xyzq(got, nx, ny, nz), fx, rtol=1e-12, atol=1e-15)

    def test_symmetry_swap_x_and_z(self, rng):
        """The update is invariant under relabelling x <-> z (velocity set
        permuted accordingly): pins the xz / z-axis links to the xy ones
        the bridge already covers."""
        nx, ny, nz = 5, 4, 6
        grid = B.open_mask(nx, ny, nz)
        grid[2, 1, 3] = B.SOLID
        grid[0, 2, 4] = B.MOVING_WALL
        wall_u = (0.03, -0.02, 0.05)
        f = random_block(rng, grid.size, np.float64)
        got = f.copy()
        oracle_for(grid, 1.3, wall_u).step(f, got)
        perm = [int(np.nonzero((L.C == (c[2], c[1], c[0])).all(1))[0][0]) for c in L.C]
        fs = to_xyzq(f, nx, ny, nz).transpose(2, 1, 0, 3)[..., perm]
        grid_s = np.ascontiguousarray(grid.transpose(2, 1, 0))
        fs_block = from_xyzq(np.ascontiguousarray(fs))
        got_s = fs_block.copy()
        oracle_for(grid_s, 1.3, (wall_u[2], wall_u[1], wall_u[0])).step(fs_block, got_s)
        back = to_xyzq(got_s, nz, ny, nx).transpose(2, 1, 0, 3)
        assert [perm[j] for j in perm] == list(range(19))  # the relabelling is an involution
        np.testing.assert_allclose(back[..., perm], to_xyzq(got, nx, ny, nz),
                                   rtol=1e-13, atol=1e-16)


# ---- 4. partition invariance -------------------------------------------------
class TestPartitionInvariance:
    def test_thread_count_never_changes_bits(self, rng):
        grid, wall_u, inlet_u = geometries3d()["channel"]
        f = random_block(rng, grid.size, np.float32)
        outs = []
        for th in (1, 3, 8):
            outs.append(oracle_for(grid, 1.6, wall_u, inlet_u, threads=th).run(
                f.copy(), f.copy(), 3))
        for o in outs[1:]:
            np.testing.assert_array_equal(outs[0], o)

    @pytest.mark.parametrize("geom", ["cavity_oblique_lid", "channel", "periodic"])
    @pytest.mark.parametrize("parts", [1, 2, 3])
    def test_slabs_equal_whole_domain_bitwise(self, geom, parts, rng):
        """P z-slabs with halo planes and 5-population exchange == 1 domain."""
        grid, wall_u, inlet_u = geometries3d()[geom]
        nx, ny, nz = grid.shape
        xp = nx + 3  # any pitch >= nx
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        f = random_block(rng, grid.size, np.float64)
        steps, omega = 4, 1.2
        want = oracle_for(grid, omega, wall_u, inlet_u).run(f.copy(), f.copy(), steps)

        dense = f.reshape(19, nz, ny, nx)
        slabs = []
        for (z0, z1) in partition(nz, parts):
            n = z1 - z0
            fl = np.ones((n + 2, ny, xp), dtype=np.uint8)
            fl[1:-1, :, :nx] = flags[z0:z1]
            fl[0, :, :nx] = flags[(z0 - 1) % nz]
            fl[-1, :, :nx] = flags[z1 % nz]
            blocks = []
            for _ in range(2):
                blk = np.full((19, n + 2, ny, xp), np.nan)
                blk[:, 1:-1, :, :nx] = dense[:, z0:z1]
                blocks.append(blk)
            slabs.append([SlabOracle(nx, ny, n, xp, fl, omega, wall_u, inlet_u), blocks, n])

        def exchange(which):
            for r, (_, blocks, n) in enumerate(slabs):
                up = slabs[(r + 1) % parts]
                dn = slabs[(r - 1) % parts]
                for q in L.UP:
                    up[1][which][q, 0] = blocks[which][q, n]
                for q in L.DOWN:
                    dn[1][which][q, dn[2] + 1] = blocks[which][q, 1]

        exchange(0)
        pre, post = 0, 1
        for _ in range(steps):
            for orc, blocks, n in slabs:
                orc.step_range(blocks[pre], blocks[post], 0, n)
                orc.open_pass_range(blocks[post], 0, n)
            exchange(post)
            pre, post = post, pre
        got = np.concatenate([blocks[pre][:, 1:-1, :, :nx] for _, blocks, _ in slabs], axis=1)
        np.testing.assert_array_equal(got.reshape(19, -1), want)
