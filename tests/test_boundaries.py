"""Flag codes, wall term and geometry builders; the 2-D sections must be
byte-identical to the reference's masks (golden vectors generated from
lb2d.boundaries, mirrors pkg/tests/test_boundaries.py)."""

import numpy as np
import pytest

from oracle.ref3d import ref3d_step
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200.boundaries import (FLUID, INLET, MOVING_WALL, OUTLET, SOLID,
                                              cavity_mask, channel_mask, cylinder_cells,
                                              disk_cells, flatten_mask, gather_cell,
                                              moving_wall_correction, open_mask,
                                              sphere_cells)
from paper_2409_16781_b200.fields import PopulationField, mask_xyz
from paper_2409_16781_b200.lattice import OPP


def test_wire_codes_are_stable(golden):
    assert (FLUID, SOLID, MOVING_WALL, INLET, OUTLET) == (0, 1, 2, 3, 4)
    assert golden["flags_codes"].tolist() == [0, 1, 2, 3, 4]
    assert sorted(B.MASK_NAMES) == [0, 1, 2, 3, 4]


class TestMovingWallCorrection:
    def test_frozen_values(self, golden):
        got = moving_wall_correction(0.0, 5, (0.1, 0.0, 0.0))
        assert got == pytest.approx(-1.0 / 60.0, rel=1e-15)
        assert got == float(golden["mw_diag"])
        # an axis link of D2Q9 (w = 1/9) is three links of D3Q19 (1/18 + 2/36):
        # their corrections add up to the reference's value (test_boundaries.py:29-31)
        total = 0.25 + sum(moving_wall_correction(0.0, i, (0.1, 0.0, 0.0)) for i in (1, 11, 14))
        assert total == pytest.approx(float(golden["mw_axis"]), rel=1e-15)

    def test_xz_diagonal_and_z_axis(self):
        assert moving_wall_correction(0.0, 11, (0.1, 0.0, 0.0)) == pytest.approx(-1 / 60, rel=1e-15)
        assert moving_wall_correction(0.0, 9, (0.0, 0.0, 0.1)) == pytest.approx(-1 / 30, rel=1e-15)

    def test_perpendicular_wall_motion_is_free(self):
        assert moving_wall_correction(0.5, 1, (0.0, 0.2, 0.3)) == 0.5

    def test_antisymmetric_in_direction(self, rng):
        for _ in range(20):
            u = tuple(rng.uniform(-0.1, 0.1, size=3))
            for i in range(1, 19):
                a = moving_wall_correction(0.0, i, u)
                b = moving_wall_correction(0.0, int(OPP[i]), u)
                assert a == pytest.approx(-b, rel=1e-12, abs=1e-18)

    def test_projected_wall_term_is_the_reference_constant(self):
        # 2-D E link = 3-D links 1, 11, 14: 1/3 + 1/6 + 1/6 = 2/3 (kernels.py:72)
        u = (0.08, 0.0, 0.0)
        total = sum(-moving_wall_correction(0.0, i, u) for i in (1, 11, 14))
        assert total == pytest.approx((2.0 / 3.0) * 0.08, rel=1e-15)


class TestMasks:
    def test_sections_equal_reference_masks(self, golden):
        for nz in (1, 3):
            m = cavity_mask(6, 5, nz, z_walls=False)
            for z in range(nz):
                np.testing.assert_array_equal(m[:, :, z], golden["mask_cavity_6x5"])
        np.testing.assert_array_equal(cavity_mask(24, 24, 2, False)[:, :, 1],
                                      golden["mask_cavity_24"])
        np.testing.assert_array_equal(channel_mask(8, 6, 2, z_walls=False)[:, :, 0],
                                      golden["mask_channel_8x6"])
        m = channel_mask(16, 12, 3, cylinder_cells(16, 12, 3, 4, 6.0, 6.0), z_walls=False)
        for z in range(3):
            np.testing.assert_array_equal(m[:, :, z], golden["mask_channel_disk"])
        np.testing.assert_array_equal(disk_cells(20, 20, 6, 10.0, 10.0), golden["disk_20"])
        np.testing.assert_array_equal(disk_cells(16, 16, 5, 8.0, 7.5), golden["disk_half"])

    def test_cavity_with_z_walls(self):
        m = cavity_mask(6, 5, 4)
        assert m.dtype == np.uint8 and m.shape == (6, 5, 4)
        assert (m[:, :, 0] == SOLID).all() and (m[:, :, -1] == SOLID).all()
        assert (m[1:-1, -1, 1:-1] == MOVING_WALL).all()
        # all twelve edges belong to the stationary walls
        assert (m[0, -1, :] == SOLID).all() and (m[-1, -1, :] == SOLID).all()
        assert (m[1:-1, 1:-1, 1:-1] == FLUID).all()
        assert np.count_nonzero(m == MOVING_WALL) == 4 * 2

    def test_channel_with_z_walls(self):
        m = channel_mask(8, 6, 5)
        assert (m[:, 0, :] == SOLID).all() and (m[:, -1, :] == SOLID).all()
        assert (m[:, :, 0] == SOLID).all() and (m[:, :, -1] == SOLID).all()
        assert (m[0, 1:-1, 1:-1] == INLET).all() and (m[-1, 1:-1, 1:-1] == OUTLET).all()
        assert (m[1:-1, 1:-1, 1:-1] == FLUID).all()

    def test_sphere(self):
        s = sphere_cells(12, 12, 12, 6, 6.0, 6.0, 6.0)
        xs, ys, zs = np.nonzero(s)
        r = np.sqrt((xs - 6.0) ** 2 + (ys - 6.0) ** 2 + (zs - 6.0) ** 2)
        assert r.max() <= 3.0 + 1e-12 and s[6, 6, 6] and not s[6, 6, 10]
        np.testing.assert_array_equal(s[1:], s[:0:-1])  # mirror symmetric about x = 6

    def test_flatten_matches_field_indexing(self):
        m = channel_mask(7, 5, 3, sphere_cells(7, 5, 3, 2, 3.0, 2.0, 1.0))
        flat = flatten_mask(m)
        f = PopulationField.alloc(7, 5, 3, np.float64)
        for x in range(7):
            for y in range(5):
                for z in range(3):
                    assert flat[f.flat(x, y, z)] == m[x, y, z]
        np.testing.assert_array_equal(mask_xyz(flat, 7, 5, 3), m)
        assert open_mask(3, 2, 2).shape == (3, 2, 2)


def test_gather_cell_matches_naive_oracle(rng):
    # test_boundaries.py:155-180: omega = 0 makes ref3d_step the bare gather
    grid = cavity_mask(6, 5, 4)
    grid[2, 2, 2] = SOLID
    wall_u = (0.07, 0.0, -0.02)
    f = PopulationField.alloc(6, 5, 4, np.float64)
    f.data[:] = rng.uniform(0.02, 1.0, size=f.data.shape)
    fx = np.stack([f.plane_xyz(i) for i in range(19)], axis=-1)
    want = ref3d_step(fx, grid, 0.0, wall_u)
    mask = flatten_mask(grid)
    for (x, y, z) in [(1, 3, 1), (4, 3, 2), (3, 2, 2), (1, 1, 1), (2, 3, 2)]:
        assert grid[x, y, z] == FLUID
        got = gather_cell(f, mask, x, y, z, wall_u)
        np.testing.assert_allclose(got, want[x, y, z], rtol=1e-14, atol=1e-17)
