"""D3Q19 lattice math: constants, the reference's known answers carried
through the z-projection, operation order and the 195-flop tally
(mirrors /root/reference/pkg/tests/test_lattice.py)."""

import numpy as np
import pytest

from oracle.ref3d import (REF_C, REF_OPP, REF_W, CountingFloat, ref_equilibrium,
                          ref_moments)
from paper_2409_16781_b200 import lattice, perfport
from paper_2409_16781_b200.lattice import (C, CS2, OPP, PROJECT_2D, W,
                                           RelaxationParams, collide, collide_cell,
                                           equilibrium, moments, omega_from_reynolds)


class TestConstants:
    def test_velocity_set(self):
        assert C.tolist() == [list(c) for c in REF_C]
        assert len({tuple(c) for c in C}) == 19
        # the reference's nine, in the reference's order (lattice.py:20-21)
        assert C[:9, :2].tolist() == [[0, 0], [1, 0], [0, 1], [-1, 0], [0, -1],
                                      [1, 1], [-1, 1], [-1, -1], [1, -1]]
        assert (C[:9, 2] == 0).all()

    def test_weights(self):
        assert W.tolist() == REF_W
        assert W.sum() == pytest.approx(1.0, abs=1e-15)

    def test_opposites(self):
        assert OPP.tolist() == REF_OPP
        for i in range(19):
            assert (C[OPP[i]] == -C[i]).all()
            assert OPP[OPP[i]] == i

    def test_weight_moments(self):
        assert np.allclose(W @ C, 0.0, atol=1e-16)
        second = np.einsum("i,ia,ib->ab", W, C.astype(float), C.astype(float))
        assert np.allclose(second, CS2 * np.eye(3), atol=1e-15)
        fourth = np.einsum("i,ia,ib,ic,id->abcd", W, *[C.astype(float)] * 4)
        d = np.eye(3)
        iso = (np.einsum("ab,cd->abcd", d, d) + np.einsum("ac,bd->abcd", d, d)
               + np.einsum("ad,bc->abcd", d, d)) / 9.0
        assert np.allclose(fourth, iso, atol=1e-15)

    def test_projection_weights_are_d2q9(self):
        # 1/3 + 2/18 = 4/9, 1/18 + 2/36 = 1/9, 1/36 = 1/36
        w2 = [W[g].sum() for g in PROJECT_2D]
        np.testing.assert_allclose(w2, [4 / 9] + [1 / 9] * 4 + [1 / 36] * 4, rtol=1e-15)
        assert sorted(np.concatenate(PROJECT_2D).tolist()) == list(range(19))

    def test_crossing_sets(self):
        assert lattice.UP.tolist() == [9, 11, 12, 15, 16]
        assert lattice.DOWN.tolist() == [10, 13, 14, 17, 18]
        assert [OPP[i] for i in lattice.UP] == [10, 13, 14, 17, 18]


class TestEquilibrium:
    def test_known_point_projects_to_reference_rationals(self, golden):
        # test_lattice.py:34-39: rho=1, u=(0.1, 0): 197/450, 133/900, ...
        feq = equilibrium(1.0, 0.1, 0.0, 0.0)
        proj = [feq[g].sum() for g in PROJECT_2D]
        expected = [197 / 450, 133 / 900, 197 / 1800, 73 / 900, 197 / 1800,
                    133 / 3600, 73 / 3600, 73 / 3600, 133 / 3600]
        np.testing.assert_allclose(proj, expected, rtol=1e-15)
        np.testing.assert_allclose(proj, golden["eq_rho1_u01"], rtol=1e-15)
        feq = equilibrium(1.2, 0.05, -0.07, 0.0)
        np.testing.assert_allclose([feq[g].sum() for g in PROJECT_2D],
                                   golden["eq_rho12_u"], rtol=1e-15)

    def test_rest_state_is_weights(self):
        np.testing.assert_allclose(equilibrium(1.0, 0.0, 0.0, 0.0), W, rtol=0)

    def test_matches_naive_reference(self, rng):
        for _ in range(200):
            rho = rng.uniform(0.5, 2.0)
            u = rng.uniform(-0.15, 0.15, size=3)
            np.testing.assert_allclose(equilibrium(rho, *u), ref_equilibrium(rho, *u),
                                       rtol=5e-15)

    def test_conserves_moments(self, rng):
        for _ in range(200):
            rho = rng.uniform(0.5, 2.0)
            u = rng.uniform(-0.2, 0.2, size=3)
            r, vx, vy, vz = moments(equilibrium(rho, *u))
            assert r == pytest.approx(rho, rel=1e-14)
            for got, want in zip((vx, vy, vz), u):
                assert got == pytest.approx(want, rel=1e-13, abs=1e-16)

    def test_batch_and_dtype(self, rng):
        rho = rng.uniform(0.9, 1.1, size=(3, 4))
        u = rng.uniform(-0.1, 0.1, size=(3, 3, 4))
        out = equilibrium(rho, *u, dtype=np.float32)
        assert out.shape == (19, 3, 4) and out.dtype == np.float32
        np.testing.assert_allclose(out, equilibrium(rho, *u), rtol=3e-6)


class TestMoments:
    def test_against_reference(self, rng):
        f = rng.uniform(0.02, 1.0, size=19)
        got = moments(f)
        want = ref_moments(list(f))
        for g, w in zip(got, want):
            assert g == pytest.approx(w, rel=1e-13)

    def test_zero_density_reports_zero_velocity(self):
        assert moments(np.zeros(19)) == (0.0, 0.0, 0.0, 0.0)
        r, ux, uy, uz = moments(np.zeros((19, 3)))
        assert (ux == 0).all() and (uy == 0).all() and (uz == 0).all()

    def test_non_finite_raises(self):
        f = np.ones(19)
        f[7] = np.nan
        with pytest.raises(ValueError, match="non-finite"):
            moments(f)


class TestCollideCell:
    def test_equals_moments_equilibrium_collide_bitwise(self, rng):
        # test_lattice.py:132-141
        for _ in range(100):
            g = rng.uniform(0.02, 1.0, size=19)
            omega = rng.uniform(0.1, 1.95)
            rho, ux, uy, uz = moments(g)
            want = collide(g, equilibrium(rho, ux, uy, uz), omega)
            got = np.array(collide_cell(list(g), omega))
            np.testing.assert_array_equal(got, want)

    def test_flop_count_is_195(self):
        ops = {"add": 0, "mul": 0, "div": 0}
        g = [CountingFloat(0.05 + 0.01 * i, ops) for i in range(19)]
        collide_cell(g, 1.3)
        assert ops["div"] == 1
        assert ops["add"] + ops["mul"] + ops["div"] == 195 == perfport.FLOPS_PER_CELL
        assert perfport.flops_per_cell() == 195

    def test_zero_density_is_safe(self):
        out = collide_cell([0.0] * 19, 1.0)
        assert all(v == 0.0 for v in out)


class TestRelaxation:
    def test_frozen_values(self, golden):
        # test_lattice.py:187-190
        assert omega_from_reynolds(1000, 0.1, 100).omega == 1.8867924528301885
        assert omega_from_reynolds(6, 0.1, 10).omega == 1.0
        assert omega_from_reynolds(1000, 0.1, 100).omega == float(golden["omega_re1000"])
        assert omega_from_reynolds(6, 0.1, 10).omega == float(golden["omega_re6"])

    def test_validation(self):
        with pytest.raises(ValueError):
            RelaxationParams.from_omega(2.0)
        with pytest.raises(ValueError):
            RelaxationParams.from_viscosity(0.0)
        with pytest.raises(ValueError):
            RelaxationParams(omega=1.0, nu=0.5)
        with pytest.raises(ValueError):
            omega_from_reynolds(0, 0.1, 10)
        with pytest.raises(ValueError, match="shape"):
            RelaxationParams.from_omega(1.0, source=np.zeros(9))
        assert RelaxationParams.from_omega(1.0, source=np.full(19, 1e-8)).has_source
        assert not RelaxationParams.from_omega(1.0).has_source


def test_c01_equilibrium_moment_exactness(rng):
    # acceptance criterion 1 (test_acceptance.py:49-63) with a third component
    rho = rng.uniform(0.5, 2.0, size=1000)
    u = rng.normal(size=(3, 1000))
    u *= rng.uniform(0.0, 0.2, size=1000) / np.linalg.norm(u, axis=0)
    got = moments(equilibrium(rho, *u))
    scale = np.maximum(1.0, np.linalg.norm(u, axis=0))
    worst = max(np.max(np.abs(got[0] - rho) / rho),
                *(np.max(np.abs(g - w) / scale) for g, w in zip(got[1:], u)))
    assert worst <= 1e-13
