"""BASELINE.json configs at their full sizes, through size-independent
properties (the oracle cannot run 512^3 in seconds) plus bounded bit-exact
windows against the oracle where it can."""

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import lattice as L
from paper_2409_16781_b200.fields import Layout, Precision

pytestmark = pytest.mark.gpu


def test_tgv256_decay_rate_and_oracle_window():
    """configs[1]: periodic Taylor-Green vortex 256^3 (the reference's exact
    2-D field extruded in z).  (a) 12 steps bit-exact against the CPU oracle
    in fp64 and fp32; (b) the fp64 decay rate of max|u| over 1000 steps
    within 5 % of the analytic 2 nu k^2 and the velocity field within 2 % L2
    of the exact solution - the reference's acceptance c03 (test_acceptance.py:81-105)."""
    import torch
    from paper_2409_16781_b200 import cases, engine
    n, nz = 256, 256
    for prec in (Precision.DOUBLE, Precision.SINGLE):
        spec = cases.CaseSpec("tgv", n, n, nz, u0=0.04, omega=1.25)
        state = cases.init(spec, prec)
        f0 = state.f_pre.data.copy()
        engine.run(state, engine.RunConfig(steps=12, precision=prec))
        want = CpuOracle(n, n, nz, state.mask, 1.25, threads=16).run(f0.copy(), f0.copy(), 12)
        np.testing.assert_array_equal(state.f_pre.data, want)
        del want, f0
    spec = cases.CaseSpec("tgv", n, n, nz, u0=0.04, omega=1.25)
    state = cases.init(spec, Precision.DOUBLE)
    nu = state.params.nu
    sess = engine.open_session(state)
    ts, amps = [], []
    for _ in range(10):
        sess.advance(100)
        ts.append(state.t)
        amps.append(sess.plan.diagnostics(sess.pre)["max_u"])
    slope = np.polyfit(ts, np.log(amps), 1)[0]
    want = -cases.tgv_decay_rate(n, nu)
    assert abs(slope - want) <= 0.05 * abs(want)
    rho, ux, uy, uz = state.macro()
    _, rx, ry, rz = cases.tgv_fields(n, 0.04, nu, state.t, nz)
    assert cases.l2_velocity_error((ux, uy), (rx, ry)) <= 0.02
    assert np.abs(uz).max() <= 1e-14
    sess.close(sync=False)
    torch.cuda.empty_cache()


def test_ldc512_fp32_properties():
    """configs[2] at full size: determinism (two runs, same bits), mass
    conservation in the closed box, never-written walls, finite fields, and
    2 z-slabs == 1 domain bitwise."""
    import torch
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    from paper_2409_16781_b200.lattice import omega_from_reynolds
    n, steps = 512, 20
    omega = omega_from_reynolds(1000.0, 0.1, n).omega
    grid = B.cavity_mask(n, n, n)
    flags = B.flatten_mask(grid)
    plan = KernelPlan(n, n, n, Layout.ROW, Precision.SINGLE, flags, omega, (0.1, 0.0, 0.0))
    np.testing.assert_array_equal(plan.device_flags(), flags)

    def fresh():
        a, b = plan.alloc(), plan.alloc()
        for q in range(19):
            a.tensor[q].fill_(float(np.float32(L.W[q])))
        b.tensor.copy_(a.tensor)
        return a, b

    a, b = fresh()
    d0 = plan.diagnostics(a)
    assert d0["fluid_cells"] == (n - 2) ** 3 and d0["nonfinite"] == 0
    res, other, _ = plan.run_steps(a, b, steps)
    d1 = plan.diagnostics(res)
    assert d1["nonfinite"] == 0
    assert abs(d1["mass"] - d0["mass"]) <= 2e-6 * d0["mass"]   # fp32 storage, 20 steps
    assert 0.0 < d1["max_u"] < 0.2 and d1["px"] > 0.0          # the lid drags fluid along +x
    # walls never written: every solid cell still holds the rest weights
    wall = res.tensor[:, 1:-1, 0, :n]
    assert all(bool((wall[q] == float(np.float32(L.W[q]))).all()) for q in range(19))
    ref = res.tensor.clone()
    del a, b, res, other
    a, b = fresh()
    res2, _, _ = plan.run_steps(a, b, steps)
    assert torch.equal(res2.tensor[:, 1:-1], ref[:, 1:-1])     # bitwise reproducible
    del a, b, res2
    plan.close()
    torch.cuda.empty_cache()

    # two z-slabs of 256 planes, halo exchange through mlb_halo_copy
    f3 = flags.reshape(n, n, n)
    slabs = []
    for (z0, z1) in slab.partition(n, 2):
        lo, hi = slab.slab_halo_flags(f3, n, n, z0, z1)
        p = KernelPlan(n, n, z1 - z0, Layout.ROW, Precision.SINGLE, f3[z0:z1], omega,
                       (0.1, 0.0, 0.0), halo_lo=lo, halo_hi=hi, slab=True)
        blocks = [p.alloc(), p.alloc()]
        for blk in blocks:
            for q in range(19):
                blk.tensor[q].fill_(float(np.float32(L.W[q])))
        slabs.append((p, blocks))
    pre, post = 0, 1
    for _ in range(steps):
        for p, blocks in slabs:
            p.step_range(blocks[pre], blocks[post], 0, p.nz)
        for r, (p, blocks) in enumerate(slabs):
            p.halo_copy(blocks[post], slabs[r - 1][1][post], face=0)
            p.halo_copy(blocks[post], slabs[(r + 1) % 2][1][post], face=1)
        pre, post = post, pre
    assert torch.equal(slabs[0][1][pre].tensor[:, 1:-1], ref[:, 1:257])
    assert torch.equal(slabs[1][1][pre].tensor[:, 1:-1], ref[:, 257:513])


def test_omega_zero_roll_256_periodic():
    """omega = 0 is the pure pull permutation (test_kernels.py:152-164) at a
    size where every thread-block shape and wrap lane is exercised."""
    import torch
    from paper_2409_16781_b200.kernels import KernelPlan
    nx, ny, nz = 256, 96, 40
    plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE,
                      B.flatten_mask(B.open_mask(nx, ny, nz)), 0.0)
    a, b = plan.alloc(), plan.alloc()
    g = torch.Generator(device="cuda").manual_seed(20240917)
    a.tensor.uniform_(0.02, 1.0, generator=g)
    b.tensor.zero_()
    plan.step(a, b)
    for q in range(19):
        src = a.tensor[q, 1:-1]
        want = torch.roll(src, shifts=(int(L.C[q][2]), int(L.C[q][1]), int(L.C[q][0])),
                          dims=(0, 1, 2))
        assert torch.equal(b.tensor[q, 1:-1], want), q


def test_channel_1024x512x512_fp32_flag_mask_path():
    """configs[4] at full size on one GPU: channel along x with solid y/z
    walls, equilibrium inlet, zero-gradient outlet and a bounce-back
    cylinder (the reference's vks geometry, z-extruded).  (a) a thin window
    of the same case, bit-exact against the oracle; (b) at full size:
    inlet / outlet semantics (engine.py:156-180) hold exactly on the device
    state, fields stay finite, solid cells untouched, and two z-slabs
    reproduce the single domain bit for bit."""
    import torch
    from paper_2409_16781_b200 import cases, engine, slab
    from paper_2409_16781_b200.kernels import KernelPlan

    # (a) oracle window: same geometry builder, 256 x 128 x 24, 15 steps
    spec = cases.CaseSpec("vks", 256, 128, 24, re=100.0, u0=0.08)
    state = cases.init(spec, Precision.SINGLE)
    f0 = state.f_pre.data.copy()
    engine.run(state, engine.RunConfig(steps=15))
    orc = CpuOracle(256, 128, 24, state.mask, state.params.omega, inlet_u=0.08, threads=16)
    np.testing.assert_array_equal(state.f_pre.data, orc.run(f0.copy(), f0.copy(), 15))
    del f0, state

    # (b) full size
    nx, ny, nz, steps = 1024, 512, 512, 12
    spec = cases.CaseSpec("vks", nx, ny, nz, re=200.0, u0=0.08)
    grid = spec.mask()
    flags = B.flatten_mask(grid)
    omega = spec.relaxation().omega
    eq = L.equilibrium(1.0, 0.08, 0.0, 0.0).astype(np.float32)          # initial fill: f64 -> f32
    eq_in = L.equilibrium(1.0, 0.08, 0.0, 0.0, dtype=np.float32)        # inlet: compute dtype

    def fresh(plan):
        a = plan.alloc()
        for q in range(19):
            a.tensor[q].fill_(float(eq[q]))
        b = plan.alloc()
        b.tensor.copy_(a.tensor)
        return a, b

    plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE, flags, omega, inlet_u=0.08)
    plan.set_passthrough(True)
    a, b = fresh(plan)
    res, _, ms = plan.run_steps(a, b, steps, timed=True)
    d = plan.diagnostics(res)
    assert d["nonfinite"] == 0 and 0.0 < d["max_u"] < 0.3
    assert d["fluid_cells"] == np.count_nonzero(flags == 0)
    t = res.tensor[:, 1:-1]                                  # (19, nz, ny, nx)
    m = torch.from_numpy(grid.transpose(2, 1, 0).copy()).cuda()   # [z][y][x]
    inlet, outlet, solid = m == B.INLET, m == B.OUTLET, m == B.SOLID
    for q in range(19):
        assert bool((t[q][inlet] == float(eq_in[q])).all())
        assert bool((t[q][..., -1][outlet[..., -1]] == t[q][..., -2][outlet[..., -1]]).all())
        assert bool((t[q][solid] == float(eq[q])).all())     # never changed
    ref = res.tensor[:, 1:-1].clone()
    print(f"channel {nx}x{ny}x{nz} fp32: {nx * ny * nz * steps / ms / 1e3:.0f} MLUPS")
    del a, b, res, t
    plan.close()
    torch.cuda.empty_cache()

    f3 = flags.reshape(nz, ny, nx)
    slabs = []
    for (z0, z1) in slab.partition(nz, 2):
        lo, hi = slab.slab_halo_flags(f3, nx, ny, z0, z1)
        p = KernelPlan(nx, ny, z1 - z0, Layout.ROW, Precision.SINGLE, f3[z0:z1], omega,
                       inlet_u=0.08, halo_lo=lo, halo_hi=hi, slab=True)
        p.set_passthrough(True)
        slabs.append((p, list(fresh(p))))
    pre, post = 0, 1
    for _ in range(steps):
        for p, blocks in slabs:
            p.step_range(blocks[pre], blocks[post], 0, p.nz)
            p.open_pass_range(blocks[post], 0, p.nz)
        for r, (p, blocks) in enumerate(slabs):
            p.halo_copy(blocks[post], slabs[r - 1][1][post], face=0)
            p.halo_copy(blocks[post], slabs[(r + 1) % 2][1][post], face=1)
        pre, post = post, pre
    assert torch.equal(slabs[0][1][pre].tensor[:, 1:-1], ref[:, :256])
    assert torch.equal(slabs[1][1][pre].tensor[:, 1:-1], ref[:, 256:])


def test_ldc1024_maximum_sizes_in_place_and_two_buffer():
    """configs[3]'s 1024^3 cavity on ONE B200.  (a) 1024 x 1024 x 512 fp32: the
    in-place run (one 41 GB block) against the two-buffer run (two blocks),
    bit for bit after an odd and an even number of steps; (b) 1024^3 fp32 in
    place (82 GB - two blocks would not fit): mass conserved in the closed box
    to rounding, fields finite, walls untouched, lid drags the fluid."""
    import torch
    from paper_2409_16781_b200.kernels import KernelPlan
    from paper_2409_16781_b200.lattice import omega_from_reynolds
    eq = L.equilibrium(1.0, 0.0, 0.0, 0.0).astype(np.float32)

    def fill(blk):
        for q in range(19):
            blk.tensor[q].fill_(float(eq[q]))

    # (a)
    nx, ny, nz = 1024, 1024, 512
    omega = omega_from_reynolds(1000.0, 0.1, nx).omega
    plan = KernelPlan(nx, ny, nz, Layout.ROW, Precision.SINGLE,
                      B.flatten_mask(B.cavity_mask(nx, ny, nz)), omega, (0.1, 0.0, 0.0))
    a, b, c = plan.alloc(), plan.alloc(), plan.alloc()
    fill(a); fill(c)
    b.tensor.copy_(a.tensor)
    plan.set_passthrough(True)
    for steps in (5, 6):
        a, b, _ = plan.run_steps(a, b, steps)
        plan.run_steps_inplace(c, steps)
        plan.normalize(c)
        assert torch.equal(a.tensor[:, 1:-1], c.tensor[:, 1:-1]), steps
    plan.close()
    del a, b, c
    torch.cuda.empty_cache()

    # (b)
    n = 1024
    plan = KernelPlan(n, n, n, Layout.ROW, Precision.SINGLE,
                      B.flatten_mask(B.cavity_mask(n, n, n)), omega, (0.1, 0.0, 0.0))
    assert plan.field_bytes > 80e9
    f = plan.alloc()
    fill(f)
    d0 = plan.diagnostics(f)
    wall = f.tensor[:, 1, :, :].clone()            # the z = 0 wall plane
    plan.run_steps_inplace(f, 11)
    plan.normalize(f)
    d1 = plan.diagnostics(f)
    assert d1["nonfinite"] == 0 and d1["fluid_cells"] == (n - 2) ** 3
    assert abs(d1["mass"] - d0["mass"]) <= 1e-6 * d0["mass"]     # fp32 storage, 11 steps
    assert 0.0 < d1["max_u"] < 0.1 and d1["px"] > 0.0            # the lid drags the fluid along +x
    assert torch.equal(f.tensor[:, 1, :, :], wall)
    plan.close()
    del f
    torch.cuda.empty_cache()


def _oracle_window(spec_args, prec, steps, inplace=False, threads=16):
    """engine.run at a BASELINE size against the CPU oracle, bitwise."""
    import torch
    from paper_2409_16781_b200 import cases, engine
    spec = cases.CaseSpec(*spec_args[0], **spec_args[1])
    state = cases.init(spec, prec)
    f0 = state.f_pre.data.copy()
    engine.run(state, engine.RunConfig(steps=steps, precision=prec, inplace=inplace))
    orc = CpuOracle(spec.nx, spec.ny, spec.nz, state.mask, state.params.omega, state.wall_u,
                    state.inlet_u, threads=threads)
    want = orc.run(f0, f0.copy(), steps)
    same = np.array_equal(state.f_pre.data, want)
    if not same:
        bad = np.argwhere(state.f_pre.data != want)
        raise AssertionError(f"{len(bad)} populations differ from the oracle, first at {bad[0]}")
    del want, f0, state
    torch.cuda.empty_cache()


def test_ldc512_fp32_oracle_window():
    """configs[2] exactly as bench.py times it - LDC 512^3 fp32, Re 1000, the
    default variant (16-byte packs), automatic prefetch distance, pass-through
    stores, cavity walls on 512-wide rows - 3 steps through engine.run against
    the CPU oracle, BITWISE (the reference's one-step / five-step kernel-vs-
    oracle tests, pkg/tests/test_kernels.py:45-79, at the headline size)."""
    _oracle_window((("ldc", 512, 512, 512), dict(re=1000.0, u0=0.1)), Precision.SINGLE, 3)


def test_ldc512_fp32_in_place_oracle_window():
    """The same configuration on ONE block (pull half, local half, pull half,
    then the swap back to the normal representation)."""
    _oracle_window((("ldc", 512, 512, 512), dict(re=1000.0, u0=0.1)), Precision.SINGLE, 3,
                   inplace=True)


def test_ldc512_fp64_oracle_window():
    _oracle_window((("ldc", 512, 512, 512), dict(re=1000.0, u0=0.1)), Precision.DOUBLE, 2)


def test_ldc1024_slab_oracle_window():
    """configs[3]'s plane shape: a 1024 x 1024 x 16 z-slab of the 1024^3 cavity
    WITH its halo planes (the slab that holds the cavity floor: solid plane
    below, fluid above), 3 steps with the halos refilled from a neighbouring
    oracle-stepped domain - i.e. the oracle runs the 1024 x 1024 x 20 piece and
    the CUDA slab must reproduce its 16 inner planes bit for bit, fed only
    through its halo planes."""
    import torch
    from paper_2409_16781_b200 import slab
    from paper_2409_16781_b200.kernels import KernelPlan
    from paper_2409_16781_b200.lattice import omega_from_reynolds
    n, nzt, steps = 1024, 24, 3
    omega = omega_from_reynolds(1000.0, 0.1, n).omega
    grid = B.cavity_mask(n, n, nzt)          # solid shell, lid on y = n-1; walls at z = 0, nzt-1
    flags = B.flatten_mask(grid).reshape(nzt, n, n)
    f = np.empty((19, nzt * n * n), dtype=np.float32)
    prng = np.random.default_rng(20240917)
    for q in range(19):   # a smooth non-trivial state: weights with a 1 % random ripple
        f[q] = (L.W[q] * (1.0 + 0.01 * prng.standard_normal(nzt * n * n))).astype(np.float32)
    orc = CpuOracle(n, n, nzt, flags, omega, (0.1, 0.0, 0.0), threads=16)
    # slab [z0, z1) of the piece; the oracle supplies the halo planes every step
    z0, z1 = 0, 16
    lo, hi = slab.slab_halo_flags(flags, n, n, z0, z1)
    plan = KernelPlan(n, n, z1 - z0, Layout.ROW, Precision.SINGLE, flags[z0:z1], omega,
                      (0.1, 0.0, 0.0), halo_lo=lo, halo_hi=hi, slab=True)
    a, b = plan.alloc(), plan.alloc()
    f4 = f.reshape(19, nzt, n, n)
    part = np.ascontiguousarray(f4[:, z0:z1]).reshape(19, -1)
    plan.upload(part, a)
    plan.upload(part, b)
    plan.set_passthrough(True)

    def fill_halos(blk, full):
        v = full.reshape(19, nzt, n, n)
        t = blk.tensor
        for q in L.UP:
            t[q, 0, :, :n] = torch.from_numpy(v[q, (z0 - 1) % nzt]).to(t.device)
        for q in L.DOWN:
            t[q, z1 - z0 + 1, :, :n] = torch.from_numpy(v[q, z1 % nzt]).to(t.device)

    cur, nxt = f, f.copy()
    pre, post = a, b
    fill_halos(pre, cur)
    for _ in range(steps):
        plan.step_open_range(pre, post, 0, z1 - z0)
        orc.step(cur, nxt)
        orc.open_pass(nxt)
        cur, nxt = nxt, cur
        pre, post = post, pre
        fill_halos(pre, cur)
    got = np.empty_like(part)
    plan.download(pre, got)
    want = np.ascontiguousarray(cur.reshape(19, nzt, n, n)[:, z0:z1]).reshape(19, -1)
    np.testing.assert_array_equal(got, want)
    plan.close()
