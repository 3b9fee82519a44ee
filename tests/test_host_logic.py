"""Host-side logic that needs no GPU: fields, cases, engine config and
state construction, perfport (mirrors the reference's test_fields.py,
test_cases.py, test_engine.py validation parts and test_perfport.py)."""

import numpy as np
import pytest

from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import cases, engine, perfport
from paper_2409_16781_b200 import lattice as L
from paper_2409_16781_b200.fields import (DeviceLayout, Layout, PopulationField, Precision,
                                          convert_precision, flat_index, flatten_xyz,
                                          mask_xyz)
from paper_2409_16781_b200.slab import partition, ring_neighbours, slab_halo_flags


class TestFields:
    def test_precision_codes_match_reference_wire_codes(self):
        assert (Precision.SINGLE.code, Precision.DOUBLE.code) == (0, 1)
        assert Precision.from_token("double") is Precision.DOUBLE
        assert Precision.from_code(0) is Precision.SINGLE
        assert Precision.MIXED1.storage == np.float16 and Precision.MIXED1.compute == np.float32
        assert Precision.from_code(2) is Precision.MIXED1  # the reference's wire code
        assert Precision.MIXED2.storage == np.float32 and Precision.MIXED2.compute == np.float64
        assert Precision.from_code(3) is Precision.MIXED2 and Precision.from_token("mixed2").code == 3
        for bad in ("mixed3", "half"):
            with pytest.raises(ValueError, match="precision"):
                Precision.from_token(bad)

    def test_layout_is_x_fastest_only(self):
        assert Layout.ROW.strides(5, 4, 3) == (1, 5, 20)
        assert flat_index(2, 3, 1, 5, 4, 3) == (1 * 4 + 3) * 5 + 2
        with pytest.raises(ValueError, match="layout"):
            Layout.from_token("col")

    def test_population_field(self, rng):
        f = PopulationField.alloc(5, 4, 3, np.float32)
        assert f.data.shape == (19, 60)
        f.set_cell(2, 1, 2, np.arange(19))
        assert f.cell(2, 1, 2).tolist() == list(range(19))
        assert f.plane_xyz(7)[2, 1, 2] == 7
        with pytest.raises(ValueError, match="shape"):
            PopulationField(np.zeros((19, 59)), 5, 4, 3)
        with pytest.raises(ValueError, match="contiguous"):
            PopulationField(np.zeros((60, 19)).T, 5, 4, 3)
        g = rng.integers(0, 5, size=(5, 4, 3)).astype(np.uint8)
        np.testing.assert_array_equal(mask_xyz(flatten_xyz(g), 5, 4, 3), g)

    def test_convert_precision_policies(self):
        big = np.array([1e300, 1.0])
        with pytest.raises(OverflowError):
            convert_precision(big, np.float32)
        out = convert_precision(big, np.float32, policy="permissive")
        assert out[0] == np.finfo(np.float32).max
        with pytest.raises(ValueError):
            convert_precision(big, np.float32, policy="lenient")

    def test_device_layout_alignment(self):
        for nx, sz in [(512, 4), (9, 8), (100, 4), (33, 8)]:
            lay = DeviceLayout(nx, 7, 5, sz)
            assert lay.xp >= nx and (lay.xp * sz) % 128 == 0
            assert (lay.plane * sz) % 128 == 0 and lay.pop == 7 * lay.plane


class TestCases:
    def test_validation(self):
        with pytest.raises(ValueError, match="unknown case"):
            cases.CaseSpec("pipe", 8, 8, 8)
        with pytest.raises(ValueError, match="too small"):
            cases.CaseSpec("ldc", 3, 8, 8)
        with pytest.raises(ValueError, match="u0"):
            cases.CaseSpec("ldc", 8, 8, 8, u0=0.5)
        with pytest.raises(ValueError, match="explicit omega"):
            cases.CaseSpec("ldc", 8, 8, 8, u0=0.0)
        with pytest.raises(ValueError, match="square"):
            cases.CaseSpec("tgv", 8, 6, 4)
        with pytest.raises(ValueError, match="multiple of 8"):
            cases.CaseSpec("vks", 64, 36, 8)
        with pytest.raises(ValueError, match="downstream"):
            cases.CaseSpec("vks", 40, 32, 8)

    def test_lengths_and_relaxation(self):
        ldc = cases.CaseSpec("ldc", 16, 100, 8, re=1000.0, u0=0.1)
        assert ldc.length == 100 and ldc.relaxation().omega == 1.8867924528301885
        vks = cases.CaseSpec("vks", 48, 32, 8)
        assert vks.diameter == 4 and vks.cyl_x == 24.0 and vks.cyl_y == 16.5
        assert vks.probe_xyz == (36, 20, 4)
        assert cases.CaseSpec("ldc", 8, 8, 8, u0=0.0, omega=1.2).relaxation().omega == 1.2

    def test_tgv_fields_equal_reference(self, golden):
        rho, ux, uy, uz = cases.tgv_fields(16, 0.04, 0.01, 7.0, nz=3)
        for z in range(3):
            np.testing.assert_array_equal(
                np.stack([rho[:, :, z], ux[:, :, z], uy[:, :, z]]), golden["tgv_fields_16"])
        assert (uz == 0).all()
        assert cases.tgv_decay_rate(64, 0.01) == pytest.approx(2 * 0.01 * (2 * np.pi / 64) ** 2)

    def test_init_states_project_onto_reference_init(self, golden):
        # cases.init of the z-extruded 2-D cases == lb2d cases.init, summed over c_z
        for name, tag, kw in (("ldc", "ldc24", dict(re=100.0, u0=0.1)),
                              ("tgv", "tgv16", dict(re=50.0, u0=0.04)),
                              ("vks", "vks48", dict(re=60.0, u0=0.1))):
            p = f"{tag}_f64_"
            nx, ny = int(golden[p + "nx"]), int(golden[p + "ny"])
            spec = cases.CaseSpec(name, nx, ny, 2, z_walls=False, **kw)
            state = cases.init(spec, Precision.DOUBLE)
            assert state.params.omega == float(golden[p + "omega"])
            np.testing.assert_array_equal(state.mask.reshape(2, -1)[1], golden[p + "mask"])
            f3 = state.f_pre.data.reshape(19, 2, -1)
            proj = np.stack([f3[g].sum(0) for g in L.PROJECT_2D])
            np.testing.assert_allclose(proj[:, 0], golden[p + "f0"], rtol=1e-14, atol=1e-17)
            assert state.f_post_ is None and state.t == 0

    def test_uniform_fast_path_equals_grid_path(self):
        m = B.cavity_mask(6, 5, 4)
        a = engine.state_from_macroscopic(1.0, 0.03, 0.0, -0.01, m, Layout.ROW, Precision.SINGLE)
        ones = np.ones((6, 5, 4))
        b = engine.state_from_macroscopic(ones, 0.03 * ones, 0 * ones, -0.01 * ones, m,
                                          Layout.ROW, Precision.SINGLE)
        np.testing.assert_array_equal(a.f_pre.data, b.f_pre.data)
        np.testing.assert_array_equal(a.f_post.data, a.f_pre.data)  # both buffers start identical

    def test_l2_velocity_error(self):
        r = (np.ones((3, 3)), np.zeros((3, 3)))
        assert cases.l2_velocity_error((1.1 * r[0], r[1]), r) == pytest.approx(0.1)
        with pytest.raises(ValueError, match="zero"):
            cases.l2_velocity_error(r, (r[1], r[1]))


class TestShedding:
    """The reference's wake analysis helpers (pkg/tests/test_cases.py:199-232)."""

    def test_zero_crossings_of_sine(self):
        from paper_2409_16781_b200.cases import zero_crossing_times
        t = np.arange(1000, dtype=np.float64)
        crossings = zero_crossing_times(np.sin(2 * np.pi * (t + 0.5) / 100.0))
        assert crossings.size == 19
        np.testing.assert_allclose(crossings[0], 49.5, rtol=1e-12)
        np.testing.assert_allclose(np.diff(crossings), 50.0, rtol=1e-12)

    def test_strouhal(self):
        from paper_2409_16781_b200.cases import strouhal
        period = 320.0
        t = np.arange(4000, dtype=np.float64)
        st, n = strouhal(0.02 * np.sin(2 * np.pi * t / period) + 1e-4 * t / 4000, 20.0, 0.1)
        assert st == pytest.approx(20.0 / (period * 0.1), rel=1e-2) and n >= 20
        t4 = np.arange(0, 4000, 4, dtype=np.float64)
        st, _ = strouhal(np.sin(2 * np.pi * t4 / period), 20.0, 0.1, sample_every=4)
        assert st == pytest.approx(20.0 / (period * 0.1), rel=1e-2)
        with pytest.raises(ValueError, match="short"):
            strouhal(np.zeros(5), 20.0, 0.1)
        with pytest.raises(ValueError, match="no shedding"):
            strouhal(np.zeros(100), 20.0, 0.1)

    def test_equal_to_the_reference_on_a_noisy_series(self):
        # values generated with the unmodified lb2d (tests/golden/make_golden.py)
        from .conftest import GOLDEN
        g = np.load(GOLDEN)
        if "strouhal_series" not in g.files:
            pytest.skip("golden file predates the shedding vectors")
        from paper_2409_16781_b200.cases import strouhal, zero_crossing_times
        np.testing.assert_array_equal(zero_crossing_times(g["strouhal_series"]),
                                      g["strouhal_crossings"])
        st, n = strouhal(g["strouhal_series"], 16.0, 0.08, sample_every=2)
        assert (st, n) == (float(g["strouhal_value"][0]), int(g["strouhal_value"][1]))


class TestEngineConfig:
    def test_schedule_and_runconfig_validation(self):
        with pytest.raises(ValueError, match="schedule"):
            engine.Schedule("diagonal")
        with pytest.raises(ValueError, match="positive"):
            engine.Schedule("tiled", 0, 4)
        with pytest.raises(ValueError, match="exceeds"):
            engine.Schedule("tiled", 64, 1).resolve(32, 8, 8, Layout.ROW)
        assert engine.Schedule("tiled", 16, 1).resolve(32, 8, 8, Layout.ROW) == (16, 1, 1)
        assert engine.Schedule().resolve(32, 8, 8, Layout.ROW) is None
        with pytest.raises(ValueError, match="steps"):
            engine.RunConfig(steps=0)
        with pytest.raises(ValueError, match="output_every"):
            engine.RunConfig(steps=1, output_every=-1)

    def test_build_plan_errors_before_touching_the_gpu(self):
        state = cases.init(cases.CaseSpec("ldc", 8, 8, 8), Precision.SINGLE)
        state.params = None
        with pytest.raises(ValueError, match="relaxation"):
            engine.build_plan(state, engine.RunConfig(steps=1))
        state.params = L.RelaxationParams.from_omega(1.0, source=np.full(19, 1e-6))
        with pytest.raises(ValueError, match="zero-source"):
            engine.build_plan(state, engine.RunConfig(steps=1))


class TestPerfport:
    def test_cost_model(self):
        assert perfport.bytes_per_cell(Precision.SINGLE) == 152
        assert perfport.bytes_per_cell("double") == 304
        assert perfport.bytes_per_cell(Precision.MIXED1) == 76
        assert perfport.arithmetic_intensity(195, 152) == pytest.approx(1.2829, rel=1e-4)
        assert perfport.mlups(512, 512, 512, 10, 0.5) == pytest.approx(2684.35456)
        with pytest.raises(ValueError):
            perfport.mlups(8, 8, 8, 1, 0.0)
        assert perfport.roofline_peak(80e3, 6551.7, 195 / 152) == pytest.approx(6551.7 * 195 / 152)
        assert perfport.roofline_efficiency(50.0, 100.0) == 0.5
        assert perfport.bandwidth_ceiling_mlups(6551.7, Precision.SINGLE) == pytest.approx(43103.3, rel=1e-5)
        assert perfport.achieved_bandwidth_gbs(37530.0, Precision.SINGLE) == pytest.approx(5704.56)

    def test_c09_roofline_reproduction(self):
        # the reference's acceptance criterion 9 (test_acceptance.py:215-224): the paper's
        # V100S row - 1.1 TB/s x AI 1.37 against 1.55 TF/s, 976 GF/s achieved = 63 %
        peak = perfport.roofline_peak(7.0e12, 1.1e12, 1.37)
        assert abs(peak - 1.55e12) / 1.55e12 <= 0.05
        assert abs(perfport.roofline_efficiency(976.0, 1550.0) - 0.63) <= 0.01


class TestSlabPartition:
    def test_partition_and_ring(self):
        assert partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
        assert partition(1024, 8)[-1] == (896, 1024)
        with pytest.raises(ValueError):
            partition(2, 3)
        assert ring_neighbours(0, 4) == (3, 1) and ring_neighbours(3, 4) == (2, 0)
        assert ring_neighbours(0, 1) == (0, 0)

    def test_halo_flags_wrap(self):
        g = np.arange(5 * 2 * 3, dtype=np.uint8).reshape(5, 2, 3) % 5
        lo, hi = slab_halo_flags(g, 3, 2, 0, 2)
        np.testing.assert_array_equal(lo, g[4])
        np.testing.assert_array_equal(hi, g[2])
        lo, hi = slab_halo_flags(g, 3, 2, 3, 5)
        np.testing.assert_array_equal(hi, g[0])

    def test_single_rank_diagnostics_combine_is_the_identity(self):
        from paper_2409_16781_b200.slab import DIAG_KEYS, combine_diagnostics
        local = dict(zip(DIAG_KEYS, [3.5, 0.1, -0.2, 0.3, 1.25, 0.07, 0.0, 42.0]))
        assert combine_diagnostics(local) == local

    def test_distributed_run_needs_a_process_group(self):
        from paper_2409_16781_b200 import cases, engine
        state = cases.init(cases.CaseSpec("ldc", 8, 8, 8), Precision.SINGLE)
        with pytest.raises(ValueError, match="process group"):
            engine.run(state, engine.RunConfig(steps=1, distributed=True))
        # auto mode without a process group is the single-GPU path: on this
        # box that means the CUDA requirement, not a distributed error
        assert engine._wants_slabs(engine.RunConfig(steps=1)) is False
        assert engine._wants_slabs(engine.RunConfig(steps=1, distributed=False)) is False
