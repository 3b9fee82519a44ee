"""The reference's acceptance gate (pkg/tests/test_acceptance.py, criteria
frozen in SPEC.md:571-584) replayed on the CUDA path.  The vortex criteria
use the reference's own 2-D field extruded along z: a z-invariant D3Q19 run
IS the D2Q9 run (z-projection), so the numbers the reference recorded for
its CPU path (pkg/test_output.txt:292-325) must come out of the GPU too."""

from dataclasses import replace

import numpy as np
import pytest

from paper_2409_16781_b200 import cases, engine
from paper_2409_16781_b200.cases import CaseSpec
from paper_2409_16781_b200.engine import RunConfig, Schedule
from paper_2409_16781_b200.fields import Precision

pytestmark = pytest.mark.gpu

# test_acceptance.py:22-26: the amplitude e-folds in exactly 2000 steps at N = 64
NU = 4096.0 / (4000.0 * 4.0 * np.pi ** 2)
OMEGA = 1.0 / (3.0 * NU + 0.5)
NZ = 4


def tgv_state(n, u0, precision=Precision.DOUBLE):
    spec = CaseSpec("tgv", n, n, NZ, u0=u0, omega=OMEGA)
    return cases.init(spec, precision), spec


def test_c02_mass_conservation():
    state, _ = tgv_state(64, 0.04)
    m0 = state.diagnostics()["mass"]
    engine.run(state, RunConfig(steps=1000, precision=Precision.DOUBLE))
    drift_tgv = abs(state.diagnostics()["mass"] - m0) / m0
    spec = CaseSpec("ldc", 48, 48, 48, u0=0.0, omega=1.0)
    state = cases.init(spec, Precision.DOUBLE)
    m0 = state.diagnostics()["mass"]
    engine.run(state, RunConfig(steps=1000, precision=Precision.DOUBLE))
    drift_ldc = abs(state.diagnostics()["mass"] - m0) / m0
    assert drift_tgv <= 1e-12 and drift_ldc <= 1e-12, (drift_tgv, drift_ldc)


def test_c03_tgv_decay_rate_and_accuracy_reproduce_the_recorded_numbers():
    state, _ = tgv_state(64, 0.04)
    sess = engine.open_session(state)
    amps = [(0, 0.04)]
    for _ in range(40):  # 2000 steps = one e-folding time
        sess.advance(50)
        _, ux, uy, uz = state.macro()
        amps.append((state.t, float(np.max(np.hypot(ux, uy)))))
        assert np.abs(uz).max() <= 1e-15
    t = np.array([a[0] for a in amps], dtype=np.float64)
    amp = np.array([a[1] for a in amps], dtype=np.float64)
    fitted = np.polyfit(t, np.log(amp), 1)[0]
    expected = -cases.tgv_decay_rate(64, state.params.nu)
    assert abs(fitted - expected) / abs(expected) <= 0.05
    _, uxr, uyr, _ = cases.tgv_fields(64, 0.04, state.params.nu, state.t, NZ)
    _, ux, uy, _ = state.macro()
    l2 = cases.l2_velocity_error((ux, uy), (uxr, uyr))
    assert l2 <= 0.02
    # pkg/test_output.txt:298 - "decay rate -5.000156e-04 ... L2 at t=tau 1.097e-03"
    assert f"{fitted:.6e}" == "-5.000156e-04"
    assert f"{l2:.3e}" == "1.097e-03"
    sess.close()


def test_c04_second_order_convergence():
    errs = {}
    for n, u0, steps in [(64, 0.04, 2000), (32, 0.08, 500)]:
        state, _ = tgv_state(n, u0)
        engine.run(state, RunConfig(steps=steps, precision=Precision.DOUBLE))
        _, uxr, uyr, _ = cases.tgv_fields(n, u0, state.params.nu, state.t, NZ)
        _, ux, uy, _ = state.macro()
        errs[n] = cases.l2_velocity_error((ux, uy), (uxr, uyr))
    ratio = errs[32] / errs[64]
    assert 3.0 <= ratio <= 5.0
    assert f"{ratio:.3f}" == "4.034"  # pkg/test_output.txt:301


def test_c05_schedule_determinism():
    variants = [("auto", RunConfig(steps=100, schedule=Schedule("auto"))),
                ("tiled(32,1,1)", RunConfig(steps=100, schedule=Schedule("tiled", 32, 1, 1))),
                ("tiled(64,4,2)", RunConfig(steps=100, schedule=Schedule("tiled", 64, 4, 2))),
                ("inplace", RunConfig(steps=100, inplace=True))]
    for precision in Precision:
        results = {}
        for label, base in variants:
            spec = CaseSpec("tgv", 64, 64, NZ, u0=0.05, omega=OMEGA)
            state = cases.init(spec, precision)
            engine.run(state, replace(base, precision=precision))
            results[label] = state.f_pre.data.copy()
        for label, data in results.items():
            np.testing.assert_array_equal(results["auto"], data, err_msg=f"{precision.token}/{label}")


def test_c06_precision_mode_error_ordering():
    fields = {}
    for precision in Precision:
        state, _ = tgv_state(32, 0.05, precision)
        engine.run(state, RunConfig(steps=500, precision=precision))
        _, ux, uy, _ = state.macro()
        assert np.isfinite(ux).all() and np.isfinite(uy).all()
        fields[precision] = (ux, uy)
    ref = fields[Precision.DOUBLE]
    err = {p: cases.l2_velocity_error(fields[p], ref) for p in Precision}
    assert err[Precision.DOUBLE] == 0.0
    # the reference's ordering (test_acceptance.py:151-172): double <= mixed2 <= single <= mixed1
    assert (err[Precision.DOUBLE] <= err[Precision.MIXED2] <= err[Precision.SINGLE]
            <= err[Precision.MIXED1])
    # same orders of magnitude as the reference recorded (pkg/test_output.txt:307:
    # mixed2 1.252e-06, single 9.114e-06, mixed1 8.935e-03); 19 stored populations round
    # differently from 9
    print(f"c06: " + ", ".join(f"{p.token} {err[p]:.3e}" for p in Precision))
    assert 1e-7 < err[Precision.MIXED2] < 1e-5
    assert 1e-6 < err[Precision.SINGLE] < 1e-4 and 1e-3 < err[Precision.MIXED1] < 5e-2


def test_c12_throughput_floor_and_runstats():
    spec = CaseSpec("ldc", 128, 128, 128, re=1000.0, u0=0.1)
    engine.run(cases.init(spec, Precision.SINGLE), RunConfig(steps=5))
    stats = engine.run(cases.init(spec, Precision.SINGLE), RunConfig(steps=25))
    assert (stats.steps, stats.nx, stats.ny, stats.nz) == (25, 128, 128, 128)
    assert stats.mlups == pytest.approx(128 ** 3 * 25 / (stats.seconds * 1e6))
    assert stats.mlups >= 5000.0  # the reference's floor is 5 MLUPS per CPU core


def test_hook_cadence_step_convenience_and_divergence():
    # test_engine.py:139-159: output at every multiple incl. the final step,
    # checkpoints only mid-run
    spec = CaseSpec("ldc", 16, 16, 12, re=50.0, u0=0.05)
    state = cases.init(spec, Precision.SINGLE)
    outs, ckpts = [], []
    engine.run(state, RunConfig(steps=12, output_every=4, checkpoint_every=6),
               on_output=lambda s: outs.append(s.t), on_checkpoint=lambda s: ckpts.append(s.t))
    assert outs == [4, 8, 12] and ckpts == [6]
    before = state.f_pre.data.copy()
    engine.step(state)                      # convenience form: host arrays are current afterwards
    assert state.t == 13 and not np.array_equal(before, state.f_pre.data)
    again = cases.init(spec, Precision.SINGLE)
    engine.run(again, RunConfig(steps=13))
    np.testing.assert_array_equal(again.f_pre.data, state.f_pre.data)
    state.f_pre.data[3, 1234] = np.nan
    with pytest.raises(engine.DivergenceError, match="divergence at step"):
        engine.run(state, RunConfig(steps=4, output_every=2))


def test_c07_vks_shedding_and_symmetry_control():
    """The reference's criterion c07 (test_acceptance.py:175-203; marked slow
    there: 40 000 steps of a 480 x 160 channel on the CPU) on the GPU path: the
    z-periodic extrusion of the same channel sheds vortices at a Strouhal number
    in [0.1, 0.3], and the symmetric control (disk on the centreline, no inflow
    perturbation) does not.  The probe series is sampled on the device every
    step; the wake analysis is the reference's (cases.strouhal)."""
    from paper_2409_16781_b200 import cases, engine
    steps = 40000

    def wake(**kw):
        spec = cases.CaseSpec("vks", 480, 160, 2, re=150.0, u0=0.1, z_walls=False, **kw)
        state = cases.init(spec, Precision.DOUBLE)
        stats = engine.run(state, engine.RunConfig(steps=steps, precision=Precision.DOUBLE),
                           probe=spec.probe_xyz)
        assert np.abs(stats.probe_samples[:, 3]).max() <= 1e-13     # z-invariant: u_z stays at rounding level
        return spec, stats.probe_series[stats.probe_series.size // 3:]

    spec, tail = wake()
    st, crossings = cases.strouhal(tail, spec.diameter, spec.u0)
    sym, tail = wake(cyl_y=(160 - 1) / 2.0, perturb=False)
    try:
        _, crossings_sym = cases.strouhal(tail, sym.diameter, sym.u0)
    except ValueError:
        crossings_sym = 0
    print(f"c07: St={st:.4f} crossings={crossings} symmetric-control crossings={crossings_sym}")
    assert 0.1 <= st <= 0.3 and crossings >= 20
    assert crossings_sym < 20 and crossings_sym < crossings


def test_bench_sweep_protocol_and_survival():
    """perfport.bench_sweep (the reference's sweep protocol, perfport.py:156-184,
    exercised there by test_perfport.py): warm-up discarded, median of reps,
    a failing job annotated instead of ending the sweep."""
    from paper_2409_16781_b200 import perfport
    from paper_2409_16781_b200.engine import RunConfig, Schedule
    good = (CaseSpec("ldc", 64, 64, 64), RunConfig(steps=20))
    inplace = (CaseSpec("ldc", 128, 32, 32), RunConfig(steps=20, inplace=True))
    bad = (CaseSpec("ldc", 16, 16, 16), RunConfig(steps=5, schedule=Schedule("tiled", 64, 1, 1)))
    seen = []
    recs = perfport.bench_sweep([good, bad, inplace], reps=3, progress=seen.append)
    assert [r.case for r in recs] == ["ldc"] * 3 and seen == recs
    assert recs[0].error == "" and recs[0].mlups > 5.0 and recs[0].seconds > 0.0
    assert recs[0].bytes_per_cell == 152 and recs[0].flops_per_cell == 195
    assert recs[0].gbs == pytest.approx(recs[0].mlups * 152e6 / 1e9)
    assert "exceeds" in recs[1].error and recs[1].mlups == 0.0
    assert recs[2].error == "" and recs[2].inplace and recs[2].mlups > 5.0
    with pytest.raises(ValueError, match="reps"):
        perfport.bench_sweep([good], reps=0)


def test_run_on_a_resident_state_keeps_the_device_steps():
    """A state made resident and advanced on the device holds its newest
    populations THERE: a following engine.run must continue from them, not
    from the stale host arrays (k + n steps == the oracle's k + n), and must
    refuse a configuration the resident session was not built for."""
    from oracle.cpu import CpuOracle
    spec = CaseSpec("ldc", 20, 18, 14, re=80.0, u0=0.08)
    for inplace in (False, True):
        state = cases.init(spec, Precision.DOUBLE)
        f0 = state.f_pre.data.copy()
        sess = engine.open_session(state, RunConfig(steps=1, precision=Precision.DOUBLE,
                                                    inplace=inplace))
        sess.advance(5)
        assert state.t == 5 and sess.host_stale
        engine.run(state, RunConfig(steps=4, precision=Precision.DOUBLE, inplace=inplace))
        assert state.t == 9
        want = CpuOracle(20, 18, 14, state.mask, state.params.omega, state.wall_u).run(
            f0.copy(), f0.copy(), 9)
        np.testing.assert_array_equal(state.f_pre.data, want)
        # host arrays current again: an edit made now IS the truth of the next run
        state.f_pre.data[:] = f0
        state.t = 0
        engine.run(state, RunConfig(steps=9, precision=Precision.DOUBLE, inplace=inplace))
        np.testing.assert_array_equal(state.f_pre.data, want)
        with pytest.raises(ValueError, match="close the session first"):
            engine.run(state, RunConfig(steps=1, precision=Precision.DOUBLE, inplace=not inplace))
        with pytest.raises(ValueError, match="close the session first"):
            engine.run(state, RunConfig(steps=1, precision=Precision.DOUBLE, inplace=inplace,
                                        schedule=Schedule("tiled", 16, 2, 2)))
        sess.close()


def test_chained_outlets_carry_the_second_block_between_sessions():
    """Where an outlet cell copies from another outlet cell the reference reads
    that cell's STALE value in fpost (engine.py:179-180), so the second buffer
    is part of the state (it is a field of the reference's SimState,
    engine.py:89).  A run cut into separate sessions - engine.step in a loop,
    run after run, the overlapped host run first - must therefore carry it:
    found by the engine-sequence fuzz (case 73), where each new session
    started its second block as a copy of the first."""
    from oracle.cpu import CpuOracle
    from paper_2409_16781_b200 import boundaries as B
    from paper_2409_16781_b200.fields import Layout, PopulationField
    from paper_2409_16781_b200.lattice import RelaxationParams
    from .helpers import geometries3d, random_block
    grid, wall_u, inlet_u = geometries3d()["open_chain"]
    nx, ny, nz = grid.shape
    mask = B.flatten_mask(grid)
    for prec in (Precision.SINGLE, Precision.MIXED2):
        f = random_block(np.random.default_rng(5), grid.size, prec.storage)
        orc = CpuOracle(nx, ny, nz, mask, 1.1, wall_u, inlet_u,
                        compute=np.float64 if prec is Precision.MIXED2 else None)
        state = engine.SimState(
            f_pre=PopulationField(f.copy(), nx, ny, nz, Layout.ROW), f_post_=None, mask=mask,
            nx=nx, ny=ny, nz=nz, layout=Layout.ROW, precision=prec,
            params=RelaxationParams.from_omega(1.1), wall_u=wall_u, inlet_u=inlet_u)
        engine.run(state, RunConfig(steps=3, precision=prec))            # (host-run path if eligible)
        for _ in range(4):
            engine.step(state)
        engine.run(state, RunConfig(steps=2, precision=prec, overlap_io=False))
        assert state.t == 9
        want = orc.run(f.copy(), f.copy(), 9)
        np.testing.assert_array_equal(state.f_pre.data, want)


def test_a_hook_that_edits_the_populations_is_loud_or_goes_through_host_edit():
    """The reference's hooks see the live host arrays (engine.py:260-265): an
    edit made in a hook is what the next step continues from.  Here the next
    step continues from the device, so a hook sees read-only views - a plain
    edit raises instead of being silently lost - and `session.host_edit()`
    is the edit that counts: the run equals the oracle's with the same edit
    at the same step."""
    from oracle.cpu import CpuOracle
    spec = CaseSpec("ldc", 20, 12, 9, re=80.0, u0=0.08)
    state = cases.init(spec, Precision.DOUBLE)
    f0 = state.f_pre.data.copy()
    cell = int(np.flatnonzero(state.mask == 0)[7])

    def bad_hook(st):
        st.f_pre.data[3, cell] = 0.5

    with pytest.raises(ValueError, match="read-only"):
        engine.run(state, RunConfig(steps=4, precision=Precision.DOUBLE, output_every=2),
                   on_output=bad_hook)
    assert state.f_pre.data.flags.writeable          # the views are gone again
    state.f_pre.data[:] = f0
    state.t = 0

    def good_hook(st):
        if st.t == 2:
            with st.session.host_edit() as s:
                s.f_pre.data[3, cell] = 0.5
            assert not st.f_pre.data.flags.writeable  # back to the hook's read-only view

    engine.run(state, RunConfig(steps=5, precision=Precision.DOUBLE, output_every=2),
               on_output=good_hook)
    orc = CpuOracle(20, 12, 9, state.mask, state.params.omega, state.wall_u)
    a, b = f0.copy(), f0.copy()
    mid = orc.run(a, b, 2)
    mid[3, cell] = 0.5
    want = orc.run(mid, b if mid is a else a, 3)
    np.testing.assert_array_equal(state.f_pre.data, want)


def test_divergence_leaves_the_diverged_populations_in_the_host_arrays():
    """engine.py:258-259 of the reference raises with the diverged populations
    in state.f_pre at the reported step; here the host arrays are synchronised
    on the way out, so `t` and the data agree."""
    spec = CaseSpec("ldc", 16, 16, 12, re=50.0, u0=0.05)
    state = cases.init(spec, Precision.SINGLE)
    state.f_pre.data[3, 1234] = np.nan
    with pytest.raises(engine.DivergenceError, match="divergence at step 2"):
        engine.run(state, RunConfig(steps=4, output_every=2))
    assert state.t == 2
    assert np.isnan(state.f_pre.data).sum() > 1     # the NaN has spread: these are step-2 data


def test_entry_points_leave_the_current_device_alone():
    """The library selects the plan's device per call and restores the caller's."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs")
    torch.cuda.set_device(0)
    spec = CaseSpec("ldc", 16, 16, 12, re=50.0, u0=0.05)
    state = cases.init(spec, Precision.SINGLE)
    engine.run(state, RunConfig(steps=3, device=1))
    assert torch.cuda.current_device() == 0


@pytest.mark.parametrize("case,prec,steps", [
    ("ldc", Precision.SINGLE, 7), ("ldc", Precision.DOUBLE, 3), ("ldc", Precision.MIXED1, 45),
    ("vks", Precision.SINGLE, 12), ("ldc", Precision.SINGLE, 93), ("vks", Precision.MIXED2, 5)])
def test_overlapped_host_run_is_the_plain_run(case, prec, steps):
    """engine.run on a host-resident state overlaps upload, steps and download
    chunk by chunk (time-skewed, mlb_run_steps_host) when the domain is closed
    in z.  Same launches per cell, so the same bits as upload / loop / download
    - compared with that path (RunConfig(overlap_io=False)) and with the CPU
    oracle, for step counts below and above one skewed sweep (40), with inlet /
    outlet faces, and with rows that are not whole 128-byte lines."""
    from oracle.cpu import CpuOracle
    spec = (CaseSpec("ldc", 256, 96, 160, re=400.0, u0=0.1) if case == "ldc"
            else CaseSpec("vks", 250, 96, 132, re=100.0, u0=0.06))
    a = cases.init(spec, prec)
    f0 = a.f_pre.data.copy()
    ra = engine.run(a, RunConfig(steps=steps, precision=prec))
    assert ra.overlapped and a.t == steps
    b = cases.init(spec, prec)
    rb = engine.run(b, RunConfig(steps=steps, precision=prec, overlap_io=False))
    assert not rb.overlapped
    np.testing.assert_array_equal(a.f_pre.data, b.f_pre.data)
    if steps <= 12:
        orc = CpuOracle(spec.nx, spec.ny, spec.nz, a.mask, a.params.omega, a.wall_u, a.inlet_u,
                        threads=8, compute=np.float64 if prec is Precision.MIXED2 else None)
        np.testing.assert_array_equal(a.f_pre.data, orc.run(f0, f0.copy(), steps))


def test_host_run_that_cannot_overlap_keeps_the_loop_timing():
    """Periodic in z (or too shallow to cut): the upload / loop / download path,
    RunStats.seconds = the update loop only, as in the reference."""
    spec = CaseSpec("tgv", 64, 64, 48, u0=0.05, omega=OMEGA)
    st = cases.init(spec, Precision.SINGLE)
    assert not engine.run(st, RunConfig(steps=5)).overlapped
    st = cases.init(CaseSpec("ldc", 32, 32, 32, re=50.0, u0=0.05), Precision.SINGLE)
    assert not engine.run(st, RunConfig(steps=5)).overlapped
