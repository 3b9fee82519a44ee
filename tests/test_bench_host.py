"""Host-side pieces of bench.py and of the overlapped host run that need no GPU:
the per-rank flag planes of every BASELINE configuration against the mask
builders, the clock-sample window, and the eligibility rule of
engine._run_host_pipelined."""

import os
import sys
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2409_16781_b200 import boundaries as B, cases, engine  # noqa: E402
from paper_2409_16781_b200.fields import Precision  # noqa: E402


@pytest.mark.parametrize("name,world", [("default", 1), ("default", 4), ("c3-weak", 2),
                                        ("c3-strong", 8), ("c4", 8)])
def test_workload_planes_are_the_mask_builders_planes(name, world):
    """bench.Workload builds a rank's flag planes without the global array; they
    must be exactly the planes of cavity_mask / channel_mask (+ the reference's
    obstacle placement, lb2d cases.py:62-75) for the whole domain."""
    wl = bench.Workload(name, world)
    # shrink the section so the global mask is cheap; the construction rule is size-blind
    wl.nx, wl.ny = wl.nx // 8, wl.ny // 8
    wl.nz = 8 * world
    wl.nzl = wl.nz // world
    if wl.case == "ldc":
        full = B.flatten_mask(B.cavity_mask(wl.nx, wl.ny, wl.nz))
    else:
        spec = cases.CaseSpec("vks", wl.nx, wl.ny, wl.nz, re=bench.CH_RE, u0=bench.CH_U0)
        full = B.flatten_mask(spec.mask())
    full = full.reshape(wl.nz, wl.ny, wl.nx)
    got = np.concatenate([wl.planes(r * wl.nzl, (r + 1) * wl.nzl) for r in range(world)])
    np.testing.assert_array_equal(got, full)
    # halo queries wrap around the periodic z axis
    np.testing.assert_array_equal(wl.planes(-1, 0)[0], full[-1])
    np.testing.assert_array_equal(wl.planes(wl.nz, wl.nz + 1)[0], full[0])


def test_workload_presets_match_baseline_configs():
    w = bench.Workload("c3-weak", 8)
    assert (w.nx, w.ny, w.nz, w.nzl, w.strong) == (1024, 1024, 1024, 128, False)
    w = bench.Workload("c3-strong", 1)
    assert (w.nz, w.nzl, w.inplace) == (1024, 1024, True)      # 2 x 82 GB do not fit one GPU
    w = bench.Workload("c3-strong", 4)
    assert (w.nz, w.nzl, w.inplace, w.strong) == (1024, 256, False, True)
    w = bench.Workload("c4", 8)
    assert (w.nx, w.ny, w.nz, w.nzl, w.case) == (1024, 512, 512, 64, "channel")
    w = bench.Workload("default", 8)
    assert (w.nz, w.nzl, w.strong) == (4096, 512, False)
    assert bench.Workload("default", 8, scaling="strong").nzl == 64
    d = bench.Workload("default", 1).describe("single")
    assert "configs[2]" in d["workload"] and d["blocks_per_gpu"] == 2
    with pytest.raises(SystemExit):
        bench.Workload("c3-strong", 3)                          # 1024 planes over 3 ranks


def test_clock_summary_uses_the_samples_inside_the_timed_region():
    s = bench.ClockSampler(0)
    t0 = time.time()
    row = lambda mhz, cap: [str(mhz), "1965", "300.0", "Not Active", "Not Active", "Not Active", cap]
    s.rows = [(t0 - 1.0, row(1200, "Not Active")), (t0 + 0.01, row(1965, "Active")),
              (t0 + 0.03, row(1950, "Not Active")), (t0 + 2.0, row(600, "Not Active"))]
    s.mark(t0, t0 + 0.05)
    out = s.summary()
    assert out["sampled"] == "timed region" and out["samples"] == 2
    assert out["sm_mhz"] == pytest.approx(1957.5) and out["reasons"] == ["sw_power_cap"]
    s.mark(t0 + 0.5, t0 + 0.51)                                  # a region with no sample inside
    assert s.summary()["sampled"].startswith("nearest samples")
    s.window = None
    assert s.summary()["samples"] == 4


def test_overlapped_host_run_eligibility():
    """engine._closed_in_z: planes 0 and nz-1 all walls AND at least four chunks of
    >= 1 MB per population (the rule mlb_run_steps_host applies)."""
    closed = cases.init(cases.CaseSpec("ldc", 256, 96, 160, re=100.0, u0=0.05), Precision.SINGLE)
    assert engine._closed_in_z(closed)
    small = cases.init(cases.CaseSpec("ldc", 32, 32, 32, re=100.0, u0=0.05), Precision.SINGLE)
    assert not engine._closed_in_z(small)                        # one chunk would hold it all
    periodic = cases.init(cases.CaseSpec("tgv", 64, 64, 48, u0=0.05, omega=1.2), Precision.SINGLE)
    assert not engine._closed_in_z(periodic)
    duct = cases.init(cases.CaseSpec("ldc", 256, 96, 160, re=100.0, u0=0.05, z_walls=False),
                      Precision.SINGLE)
    assert not engine._closed_in_z(duct)                         # periodic in z: the wrap is live
