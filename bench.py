#!/usr/bin/env python
"""bench.py - MLUPS of the D3Q19 BGK time-step loop on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config default|c3-weak|c3-strong|c4]

Workloads (BASELINE.json `configs`):
  default    configs[2], the one the metric is quoted on: lid-driven cavity,
             512^3 cells PER GPU, fp32, Re 1000, u0 0.1.  With N > 1 the
             cavity is 512 x 512 x 512N in N z-slabs (weak scaling; `--scaling
             strong` splits the 512^3 instead).
  c3-weak    configs[3] weak: cavity 1024 x 1024 x 128 per GPU (8 GPUs = 1024^3).
  c3-strong  configs[3] strong: the fixed 1024^3 cavity; in place (one block,
             82 GB) on one GPU, two blocks per rank from two GPUs on.
  c4         configs[4]: channel 1024 x 512 x 512 past a bounce-back cylinder,
             inlet / outlet faces, split over the N ranks.
With N > 1 (launched under torch.distributed.run, one rank per GPU) the
domain is cut into z-slabs; only the 5 populations that cross a face are
exchanged, stored straight into the neighbour's halo planes by the fused
kernel over CUDA-IPC peer memory (NCCL send/recv as the fallback).  Before
anything is timed at N > 1 a PREFLIGHT runs small cavity + channel cases
through the very runner that will be timed and compares the gathered result
BITWISE with the CPU oracle; the bench aborts otherwise.

One "step" is one lattice time step: the fused pull-stream + BGK collide
kernel over all cells (plus the open-boundary pass and the halo exchange).
MLUPS counts ALL cells, solid included, like the reference (lb2d
perfport.py:55-61, engine.py:270-271).

The one JSON line carries
  value      device-timed whole-job MLUPS, populations resident in HBM;
             CUDA events on the launching stream, max over ranks;
  e2e        the same K steps through the public host API
             (`engine.run` on a host-resident state in pinned memory):
             H2D of the populations + flags, K steps, D2H of the result,
             all inside the timed region;
  roofline   the fused kernel against the measured HBM bandwidth
             (MEASURED_PEAKS.json): algorithmic bytes 2 x 19 x 4 B per
             update (lb2d perfport.py:40-45 with Q = 19); `traffic` is the
             ncu DRAM byte count recorded for THIS build (profiles/traffic.json
             entries carry the library's build id), else null;
  parity     (N = 1) the timed configuration itself against the CPU oracle:
             the first steps of the benchmark's own initial state, full size,
             compared bitwise;
  cpu_baseline  the same oracle steps, timed: a C/OpenMP port of the
             reference's algorithm on all host cores;
  cpu_baseline_ref2d  the UNMODIFIED reference (lb2d, numba D2Q9, installed
             into baseline/_ref) on its own 2-D cavity, as context;
  extra      (N = 1 by default, `--extra` at N > 1) short device-timed runs
             of the other BASELINE configurations: c3-strong, c3-weak, c4, and
             at N = 1 also c0 (64^3 fp64, L2-resident, loop replayed from a CUDA
             graph) and c1 (the periodic 256^3 box, fp64 and fp32).

`--impl reference` times the CPU port alone, on the same config, each step
a bounded z-slice of the cavity so the run ends within a few minutes.  The
oracle is used here as the checker and as the measured CPU arm only; it is
never on the GPU path.
"""

import argparse
import json
import os
import signal
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RE, U0 = 1000.0, 0.1
CH_RE, CH_U0 = 200.0, 0.08
METRIC = "MLUPS (D3Q19 BGK)"
PREC_NAME = {"single": "fp32", "double": "fp64", "mixed1": "fp16 storage / fp32 compute",
             "mixed2": "fp32 storage / fp64 compute"}
PREC_BYTES = {"single": 4, "double": 8, "mixed1": 2, "mixed2": 4}
PREC_DTYPE = {"single": "f32", "double": "f64", "mixed1": "f16 storage, f32 compute",
              "mixed2": "f32 storage, f64 compute"}
PREC_TAG = {"single": "f32", "double": "f64", "mixed1": "f16", "mixed2": "m2"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="default", choices=["default", "c0", "c1", "c3-weak", "c3-strong", "c4"],
                    help="which BASELINE.json configuration to time (see the module docstring)")
    ap.add_argument("--edge", "--n", dest="n", type=int, default=0,
                    help="default config only: override the edge length (debug)")
    ap.add_argument("--precision", default="single", choices=["single", "double", "mixed1", "mixed2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="N = 1: skip the short runs of the other BASELINE configurations")
    ap.add_argument("--extra", action="store_true",
                    help="N > 1: also time c3-weak / c3-strong / c4 (20 steps each) into `extra`")
    ap.add_argument("--no-preflight", action="store_true", help="N > 1: skip the bitwise preflight")
    ap.add_argument("--preflight-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--force-slab", action="store_true",
                    help="run the z-slab driver (halo planes, boundary-first overlap) even on 1 GPU")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="halo exchange of the z-slab run: 'peer' = stores into the neighbours' halo "
                         "planes from inside the fused kernel over CUDA-IPC-mapped peer memory "
                         "(default; falls back to 'nccl' if the mapping cannot be set up), "
                         "'nccl' = torch.distributed send/recv")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="default config, N > 1: 'weak' = 512^3 cells per GPU (what the driver's "
                         "scaling run measures), 'strong' = the 512^3 domain split into N z-slabs")
    ap.add_argument("--inplace", action="store_true",
                    help="the in-place update (one population block per GPU instead of two; same "
                         "arithmetic and traffic)")
    ap.add_argument("--python-loop", action="store_true",
                    help="z-slab runs: drive the per-step schedule from Python instead of the "
                         "library's one-call loop (mlb_slab_run_steps) - for A/B runs")
    ap.add_argument("--share-gpu", action="store_true",
                    help="debug, not a benchmark: all ranks use device 0 with a gloo control plane, so "
                         "a one-GPU box can drive the N > 1 code path (peer ring across processes)")
    ap.add_argument("--variant", type=int, default=0, help="kernel variant (tuning; see mlb_plan_set_variant)")
    return ap.parse_args()


# --------------------------------------------------------------------------
# workloads: global domain, per-plane flags, initial populations
class Workload:
    """One BASELINE configuration: the global domain, how it is cut, and how a
    rank builds its part without materialising the global arrays."""

    def __init__(self, name, world, n=0, scaling="weak", inplace=False):
        self.name, self.world = name, world
        self.inplace = inplace
        if name == "default":
            e = n or 512
            self.case, self.nx, self.ny = "ldc", e, e
            self.strong = scaling == "strong" and world > 1
            self.nz = e if (self.strong or world == 1) else e * world
            self.label = "configs[2]"
        elif name == "c0":
            # configs[0]: the reference's CPU-runnable case (parity config; here: throughput)
            self.case, self.nx, self.ny, self.nz = "ldc", 64, 64, 64
            self.strong, self.label = True, "configs[0]"
        elif name == "c1":
            # configs[1]: periodic box of the Taylor-Green case (all fluid, no walls)
            self.case, self.nx, self.ny, self.nz = "periodic", 256, 256, 256
            self.strong, self.label = True, "configs[1] geometry"
        elif name == "c3-weak":
            self.case, self.nx, self.ny, self.nz = "ldc", 1024, 1024, 128 * world
            self.strong, self.label = False, "configs[3] weak"
        elif name == "c3-strong":
            self.case, self.nx, self.ny, self.nz = "ldc", 1024, 1024, 1024
            self.strong, self.label = True, "configs[3] strong"
            if world == 1:
                self.inplace = True     # two blocks of 82 GB do not fit one GPU
        elif name == "c4":
            self.case, self.nx, self.ny, self.nz = "channel", 1024, 512, 512
            self.strong, self.label = True, "configs[4]"
        else:
            raise ValueError(name)
        if self.nz % world:
            raise SystemExit(f"{name}: {self.nz} planes do not split evenly over {world} ranks")
        self.nzl = self.nz // world
        if self.case in ("ldc", "periodic"):
            self.re, self.u0 = (100.0 if name == "c0" else RE), U0
            self.wall_u, self.inlet_u, self.length = (U0, 0.0, 0.0), 0.0, self.ny
        else:
            self.re, self.u0 = CH_RE, CH_U0
            self.wall_u, self.inlet_u, self.length = (0.0, 0.0, 0.0), CH_U0, self.ny // 8

    @property
    def omega(self):
        from paper_2409_16781_b200.lattice import omega_from_reynolds
        return omega_from_reynolds(self.re, self.u0, self.length).omega

    def _section(self):
        """[y][x] flags of a plane strictly inside the z walls."""
        import numpy as np
        from paper_2409_16781_b200 import boundaries as B
        if self.case == "ldc":
            m = B.cavity_mask(self.nx, self.ny, 1, z_walls=False)
        elif self.case == "periodic":
            m = B.open_mask(self.nx, self.ny, 1)
        else:
            d = self.ny // 8    # the reference's obstacle placement (lb2d cases.py:62-75)
            obs = B.cylinder_cells(self.nx, self.ny, 1, d, 6.0 * d, self.ny / 2 + 0.5)
            m = B.channel_mask(self.nx, self.ny, 1, obs, z_walls=False)
        return np.ascontiguousarray(m[:, :, 0].T)

    def planes(self, z0, z1):
        """Dense [z1-z0][ny][nx] flags of global planes z0..z1-1 (periodic in z):
        what boundaries.cavity_mask / channel_mask give for the whole domain."""
        import numpy as np
        from paper_2409_16781_b200 import boundaries as B
        sec = self._section()
        out = np.empty((z1 - z0, self.ny, self.nx), dtype=np.uint8)
        for k, z in enumerate(range(z0, z1)):
            zz = z % self.nz
            out[k] = B.SOLID if (zz in (0, self.nz - 1) and self.case != "periodic") else sec
        return out

    def init_values(self, dtype):
        """The 19 population values every cell starts from (uniform state)."""
        import numpy as np
        from paper_2409_16781_b200 import lattice as L
        if self.case in ("ldc", "periodic"):
            return np.asarray(L.W, dtype=np.float64).astype(dtype)
        return L.equilibrium(1.0, self.u0, 0.0, 0.0).astype(dtype)

    def describe(self, prec, transport=None):
        size = f"{self.nx}^3" if self.nx == self.ny == self.nz else f"{self.nx}x{self.ny}x{self.nz}"
        what = ("lid-driven cavity" if self.case == "ldc"
                else "periodic box (the Taylor-Green case's geometry, uniform state)"
                if self.case == "periodic"
                else "channel past a bounce-back cylinder (inlet / outlet faces)")
        scal = f", z-slab {'strong' if self.strong else 'weak'} scaling" if self.world > 1 else ""
        cfg = {
            "workload": f"D3Q19 BGK {what} {size} {PREC_NAME[prec]} (BASELINE.json {self.label}{scal})",
            "nx": self.nx, "ny": self.ny, "nz_per_gpu": self.nzl, "nz_global": self.nz,
            "re": self.re, "u0": self.u0, "omega": self.omega,
            "decomposition": (f"{self.world} z-slab(s), 5-population halos" if self.world > 1
                              else "single GPU"),
            "blocks_per_gpu": 1 if self.inplace else 2,
            "l2_policy": (
                f"inputs exceed L2: {'one population block' if self.inplace else 'two population blocks'} of "
                f"{19 * self.nx * self.ny * self.nzl * PREC_BYTES[prec] / 1e9:.1f} GB per GPU vs 126 MB L2"
                if 19 * self.nx * self.ny * self.nzl * PREC_BYTES[prec] * (1 if self.inplace else 2) > 126e6
                else f"NOT flushed: the whole state ({19 * self.nx * self.ny * self.nzl * PREC_BYTES[prec] * (1 if self.inplace else 2) / 1e6:.0f} MB) "
                     f"fits the 126 MB L2 - a small-domain figure, not an HBM figure"),
        }
        if transport:
            cfg["halo_transport"] = transport
        return cfg


# --------------------------------------------------------------------------
# clocks: sample nvidia-smi during the timed region (B200_PROFILING.md)
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None
        self.window = None   # (t0, t1) of the timed region, host clock

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self):
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows, where = [r for _, r in self.rows], "whole run (sampler started before the warm-up)"
        if self.window is not None:
            # samples taken while the timed region ran (a sample reports the state a
            # few ms before it is printed); a region shorter than the sampling
            # period may hold none: then the samples closest around it
            t0, t1 = self.window
            inside = [r for t, r in self.rows if t0 <= t <= t1 + 0.03]
            if inside:
                rows, where = inside, "timed region"
            else:
                near = sorted(self.rows, key=lambda tr: min(abs(tr[0] - t0), abs(tr[0] - t1)))[:3]
                if near:
                    rows, where = [r for _, r in near], "nearest samples around the timed region"
        for r in rows:
            if len(r) < 7:
                continue
            try:
                sm.append(float(r[0])); mx.append(float(r[1]))
            except ValueError:
                continue
            try:
                pw.append(float(r[2]))
            except ValueError:
                pass
            for name, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm), "sampled": where,
                "power_w": statistics.median(pw) if pw else None}


# --------------------------------------------------------------------------
# CPU arms
def _np_dtype(prec):
    import numpy as np
    return {"single": np.float32, "double": np.float64, "mixed1": np.float16,
            "mixed2": np.float32}[prec]


def cpu_arm(n, prec, steps, warmup, budget_s):
    """Time the CPU port of the reference algorithm (the oracle, OpenMP over
    all host cores) on a bounded z-slice of the cavity."""
    import numpy as np
    from oracle.cpu import CpuOracle
    from paper_2409_16781_b200 import boundaries as B
    from paper_2409_16781_b200.lattice import W, omega_from_reynolds
    cores = os.cpu_count() or 1
    dtype = _np_dtype(prec)
    omega = omega_from_reynolds(RE, U0, n).omega

    def make(nz):
        mask = B.flatten_mask(B.cavity_mask(n, n, nz))
        f = np.empty((19, n * n * nz), dtype=dtype)
        for q in range(19):
            f[q].fill(W[q])
        return CpuOracle(n, n, nz, mask, omega, (U0, 0.0, 0.0), threads=cores,
                         compute=np.float64 if prec == "mixed2" else None), f, f.copy()

    # calibrate on a thin slice, then size the sample to the time budget
    orc, a, b = make(8)
    orc.step(a, b)
    t0 = time.perf_counter(); orc.step(b, a); dt = time.perf_counter() - t0
    rate = n * n * 8 / dt
    nz = int(rate * budget_s / ((steps + warmup) * n * n))
    nz = max(32, min(n, nz))
    orc, a, b = make(nz)
    for _ in range(warmup):
        orc.step(a, b); a, b = b, a
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.step(a, b); a, b = b, a
    dt = time.perf_counter() - t0
    mlups = n * n * nz * steps / dt / 1e6
    return {"value": mlups, "unit": "MLUPS", "cores": cores, "kind": "port",
            "sample": f"{n}x{n}x{nz} z-slice of the cavity, {steps} steps after {warmup} warm-up, "
                      f"{PREC_NAME[prec]}, C/OpenMP port of the reference "
                      f"algorithm (oracle/d3q19_oracle.c), {cores} threads"}, dt / steps * 1e3


def parity_and_cpu_baseline(wl, prec, state_mask, f_init, gpu_after, steps):
    """The timed configuration against the oracle, at full size: `steps` oracle
    steps from the benchmark's own initial state `f_init` (timed: this is also
    the cpu_baseline sample), compared bitwise with `gpu_after(steps)`, the
    populations the GPU path holds after the same number of steps."""
    import numpy as np
    from oracle.cpu import CpuOracle
    cores = os.cpu_count() or 1
    orc = CpuOracle(wl.nx, wl.ny, wl.nz, state_mask, wl.omega, wl.wall_u, wl.inlet_u,
                    threads=cores, compute=np.float64 if prec == "mixed2" else None)
    a, b = f_init, f_init.copy()
    orc.step(a, b); orc.open_pass(b); a, b = b, a          # warm-up (page faults of `b`)
    t0 = time.perf_counter()
    for _ in range(steps - 1):
        orc.step(a, b); orc.open_pass(b); a, b = b, a
    dt = time.perf_counter() - t0
    del b
    got = gpu_after(steps)
    same = bool(np.array_equal(got, a))
    cells = wl.nx * wl.ny * wl.nz
    parity = {"against": "CPU oracle (oracle/d3q19_oracle.c), same initial state, full size",
              "size": f"{wl.nx}x{wl.ny}x{wl.nz}", "steps": steps,
              "result": "bitwise" if same else "MISMATCH",
              "populations_compared": int(a.size)}
    if not same:
        parity["differing"] = int(np.count_nonzero(got != a))
    base = {"value": cells * (steps - 1) / dt / 1e6, "unit": "MLUPS", "cores": cores, "kind": "port",
            "sample": f"the whole {wl.nx}x{wl.ny}x{wl.nz} domain, {steps - 1} steps after 1 warm-up, "
                      f"{PREC_NAME[prec]}, C/OpenMP port of the reference algorithm "
                      f"(oracle/d3q19_oracle.c), {cores} threads; the same steps are the parity check"}
    return parity, base


def ref2d_arm():
    """The UNMODIFIED reference (lb2d, numba backend) on its own 2-D D2Q9 cavity,
    from baseline/_ref (installed by tools/install_reference.sh; pure Python, so it
    travels to the GPU box).  Context only: a different lattice (9 velocities,
    72 B per update in fp32)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lb2d")):
        return {"unavailable": "baseline/_ref/lb2d is not installed (tools/install_reference.sh)"}
    code = r"""
import json, os, sys, time
sys.path.insert(0, sys.argv[1])
os.environ.setdefault("LB2D_BACKEND", "numba")
from lb2d import cases, engine, kernels
from lb2d.fields import Layout, Precision
import numba
out = {"backend": kernels.BACKEND, "threads": numba.get_num_threads(), "cores": os.cpu_count(), "runs": []}
for n, steps in ((512, 100), (4096, 10)):
    spec = cases.CaseSpec("ldc", n, n, re=1000.0, u0=0.1)
    best = 0.0
    for rep in range(3):
        st = cases.init(spec, Precision.SINGLE, Layout.COL)
        if rep == 0:
            engine.run(st, engine.RunConfig(steps=2, precision=Precision.SINGLE, layout=Layout.COL, threads=os.cpu_count()))
        r = engine.run(st, engine.RunConfig(steps=steps, precision=Precision.SINGLE, layout=Layout.COL, threads=os.cpu_count()))
        best = max(best, r.mlups)
    out["runs"].append({"case": f"LDC {n}^2 fp32 col, {steps} steps, best of 3", "mlups": best})
print(json.dumps(out))
"""
    try:
        res = subprocess.run([sys.executable, "-c", code, ref], capture_output=True, text=True,
                             timeout=240)
        if res.returncode != 0:
            return {"unavailable": (res.stderr.strip().splitlines() or ["failed"])[-1][:200]}
        out = json.loads(res.stdout.strip().splitlines()[-1])
    except Exception as exc:   # numba missing on the box, time-out, ...
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    out.update({"kind": "reference", "unit": "MLUPS (D2Q9, 2-D)",
                "what": "unmodified lb2d (pkg/src/lb2d/engine.py:218-275), numba backend, all host cores"})
    return out


# --------------------------------------------------------------------------
def preflight(args, rank, world, device, fdev):
    """Small cavity + channel through the very runners that get timed - same
    transport, same one-call loop, two blocks and in place, fp32 and fp64 -
    gathered to rank 0 and compared BITWISE with the CPU oracle (the reference's
    partition-independence bar, pkg/tests/test_kernels.py:107-126).  Returns a
    record whose "result" is "bitwise" or names the first case that differs."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from oracle.cpu import CpuOracle
    from paper_2409_16781_b200 import boundaries as B, slab
    from paper_2409_16781_b200.fields import Layout, Precision
    from paper_2409_16781_b200.kernels import KernelPlan
    # (nx = 128: the pack kernels the timed run uses are the automatic choice from there on)
    nx, ny, nz, steps = 128, 40, 8 * world, 7
    cav = B.cavity_mask(nx, ny, nz)
    cav[20:24, 10:14, 3:nz - 2] = B.SOLID
    chan = B.channel_mask(nx, ny, nz, B.cylinder_cells(nx, ny, nz, 8, 40.0, 20.5))
    cases_ = [("cavity", cav, (0.07, 0.0, 0.0), 0.0), ("channel", chan, (0.0, 0.0, 0.0), 0.05)]
    transports, skipped = set(), set()
    n = 0
    for name, grid, wall_u, inlet_u in cases_:
        flags = B.flatten_mask(grid).reshape(nz, ny, nx)
        for prec in (Precision.SINGLE, Precision.DOUBLE):
            f = np.ascontiguousarray(np.random.default_rng(20240917).uniform(
                0.02, 1.0, size=(19, nz * ny * nx)).astype(prec.storage))
            z0, z1 = slab.partition(nz, world)[rank]
            lo, hi = slab.slab_halo_flags(flags, nx, ny, z0, z1)
            part = np.ascontiguousarray(f.reshape(19, nz, ny, nx)[:, z0:z1]).reshape(19, -1)
            for inplace in ((False, True) if args.transport == "peer" else (False,)):
                plan = KernelPlan(nx, ny, z1 - z0, Layout.ROW, prec, flags[z0:z1], 1.3, wall_u,
                                  inlet_u=inlet_u, device=device.index, halo_lo=lo, halo_hi=hi,
                                  slab=True)
                a = plan.alloc()
                plan.upload(part, a)
                if inplace:
                    try:
                        runner = slab.open_inplace_runner(plan, a, rank, world)
                    except RuntimeError as exc:
                        # no peer memory between the ranks (every rank raises alike): the
                        # in-place slabs cannot run here at all; the two-block run still can
                        skipped.add(f"in place: {exc}"[:160])
                        plan.close()
                        continue
                    runner.c_loop = not args.python_loop
                    runner.run_inplace(a, steps)
                    runner.normalize(a)
                    newest, tr = a, "peer"
                else:
                    b = plan.alloc()
                    b.tensor.copy_(a.tensor)
                    try:
                        plan.set_passthrough(True)
                    except ValueError:
                        plan.set_passthrough(False)
                    runner, tr = slab.open_runner(plan, a, b, rank, world, transport=args.transport)
                    runner.c_loop = not args.python_loop
                    newest, _ = runner.run(a, b, steps)
                    runner.finish()
                transports.add(tr)
                got = np.empty_like(part)
                plan.download(newest, got)
                if runner.ring is not None:
                    runner.ring.close()
                plan.close()
                parts = [None] * world
                if world > 1:
                    dist.all_gather_object(parts, got)
                else:
                    parts = [got]
                ok = True
                if rank == 0:
                    whole = np.concatenate([p.reshape(19, -1, ny, nx) for p in parts], axis=1)
                    want = CpuOracle(nx, ny, nz, flags, 1.3, wall_u, inlet_u, threads=4).run(
                        f.copy(), f.copy(), steps)
                    ok = bool(np.array_equal(whole.reshape(19, -1), want))
                flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                    device=device if fdev is not None else "cpu")
                if world > 1:
                    dist.broadcast(flag, src=0)
                if not bool(flag.item()):
                    return {"result": f"MISMATCH: {name} {prec.token} "
                                      f"{'in place' if inplace else 'two blocks'} over {world} slabs "
                                      f"(halo transport {tr}) differs from the CPU oracle",
                            "cases": n, "transports": sorted(transports)}
                n += 1
    return {"result": "bitwise", "cases": n, "transports": sorted(transports),
            "skipped": sorted(skipped),
            "what": f"cavity + channel {nx}x{ny}x{nz}, fp32 + fp64, {steps} steps, two blocks + in place, "
                    f"{world} z-slab(s), vs the CPU oracle"}


def preflight_child(args):
    """`bench.py --preflight-child`: one rank of the preflight in its OWN process
    and process group (rendezvous on MASTER_PORT of its environment), so that a
    protocol problem on hardware this code has never met - a peer mapping that
    cannot be made, a counter that never arrives - costs a child process and not
    the benchmark.  Prints one JSON line."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    fdev = None if args.share_gpu else device
    if world > 1:
        init = f"tcp://{os.environ.get('MASTER_ADDR', '127.0.0.1')}:{os.environ['MASTER_PORT']}"
        if args.share_gpu:
            dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", init_method=init, rank=rank, world_size=world,
                                    device_id=device)
    try:
        rec = preflight(args, rank, world, device, fdev)
        if os.environ.get("MLB_PREFLIGHT_FAIL") == args.transport:   # (test hook for the fallback)
            rec = {"result": f"MISMATCH: forced by MLB_PREFLIGHT_FAIL={args.transport}"}
    except BaseException as exc:     # incl. SystemExit from the library layers
        rec = {"result": f"ERROR: {type(exc).__name__}: {exc}"[:300]}
    print(json.dumps(rec), flush=True)
    if world > 1:
        try:
            dist.destroy_process_group()
        except Exception:
            pass
    return 0


def preflight_guarded(args, world, timeout_s=240):
    """Run this rank's part of the preflight in a child process with a hard
    time limit; returns its record (result "bitwise", "MISMATCH ...", "ERROR ..."
    or "TIMEOUT")."""
    env = dict(os.environ)
    env["MASTER_PORT"] = str(20000 + (int(env.get("MASTER_PORT", "29500")) + 17) % 40000)
    env["TORCHELASTIC_USE_AGENT_STORE"] = "False"
    cmd = [sys.executable, os.path.abspath(__file__), "--preflight-child", "--gpus", str(world),
           "--transport", args.transport]
    if args.share_gpu:
        cmd.append("--share-gpu")
    if args.python_loop:
        cmd.append("--python-loop")
    try:
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout_s)
    except subprocess.TimeoutExpired:
        return {"result": f"TIMEOUT: the preflight did not finish within {timeout_s} s"}
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    if res.returncode != 0 or not lines:
        tail = (res.stderr.strip().splitlines() or ["no output"])[-1]
        return {"result": f"ERROR: preflight child exited with {res.returncode}: {tail}"[:300]}
    return json.loads(lines[-1])


def run_device(wl, args, prec_tok, rank, world, device, fdev, steps, warmup, clocks=False):
    """Device-timed run of one workload: W warm-up steps, then exactly K steps
    bracketed by barrier + synchronize, CUDA events, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2409_16781_b200 import _cabi, slab
    from paper_2409_16781_b200.fields import Layout, Precision
    from paper_2409_16781_b200.kernels import KernelPlan
    prec = Precision.from_token(prec_tok)
    nx, ny, nzl = wl.nx, wl.ny, wl.nzl
    slab_mode = world > 1 or args.force_slab

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    z0 = rank * nzl
    flags = wl.planes(z0, z0 + nzl)
    if slab_mode:
        lo, hi = wl.planes(z0 - 1, z0)[0], wl.planes(z0 + nzl, z0 + nzl + 1)[0]
        plan = KernelPlan(nx, ny, nzl, Layout.ROW, prec, flags, wl.omega, wl.wall_u,
                          inlet_u=wl.inlet_u, device=device.index, halo_lo=lo, halo_hi=hi, slab=True)
    else:
        plan = KernelPlan(nx, ny, nzl, Layout.ROW, prec, flags, wl.omega, wl.wall_u,
                          inlet_u=wl.inlet_u, device=device.index)
    if args.variant:
        plan.set_variant(args.variant)
    kernel_name = plan.kernel_name if not wl.inplace else \
        "mlb::aa_pull_vec_kernel + mlb::aa_local_vec_kernel (alternating)"
    vals = wl.init_values(prec.storage)
    a = plan.alloc()
    for q in range(19):
        a.tensor[q].fill_(float(vals[q]))
    runner, transport, b = None, None, None
    if wl.inplace:
        if slab_mode:
            runner, transport = slab.open_inplace_runner(plan, a, rank, world), "peer"
    else:
        b = plan.alloc()
        b.tensor.copy_(a.tensor)
        try:
            plan.set_passthrough(True)   # both blocks identical: what engine.Session establishes
        except ValueError:
            plan.set_passthrough(False)
        if slab_mode:
            runner, transport = slab.open_runner(plan, a, b, rank, world, transport=args.transport)
    if runner is not None:
        runner.c_loop = not args.python_loop

    def advance(x, y, k):
        if wl.inplace:
            if runner is None:
                plan.run_steps_inplace(x, k)
            else:
                runner.run_inplace(x, k)
            return x, y
        if runner is None:
            newest, other, _ = plan.run_steps(x, y, k)
            return newest, other
        return runner.run(x, y, k)

    def settle(x):
        """Pushes landed; in place: the block back in the normal representation."""
        if runner is not None and wl.inplace:
            runner.normalize(x)
        elif runner is not None:
            runner.finish()
        elif wl.inplace:
            plan.normalize(x)

    sampler = ClockSampler(device.index) if clocks else None
    if sampler:
        sampler.__enter__()      # nvidia-smi takes a while to start: before the warm-up
    a, b = advance(a, b, warmup)
    if not wl.inplace:
        settle(a)
    elif runner is not None:
        runner.finish()
    barrier()
    if runner is not None and runner.ring is not None and not wl.inplace:
        # the fused exchange against the plain one, on live data: the halos the
        # kernels stored into this rank must be the planes send/recv delivers
        if not slab.halos_match_send_recv(plan, a, rank, world):
            raise SystemExit("bench: fused peer-store halos differ from the send/recv exchange")
    launches0 = _cabi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        if sampler:
            time.sleep(0.3)      # the sampler's first rows, with the GPU idle
        w0 = time.time()
        e0.record()
        t_host = time.perf_counter()
        a, b = advance(a, b, steps)
        host_enqueue = time.perf_counter() - t_host
        e1.record()
        if runner is not None:
            runner.finish()
        barrier()
        if sampler:
            sampler.mark(w0, time.time())
            time.sleep(0.05)
    finally:
        if sampler:
            sampler.__exit__(None, None, None)
    settle(a)
    launches = _cabi.launch_count() - launches0
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    nl = torch.tensor([launches], dtype=torch.int64, device=device)
    if world > 1 and fdev is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    elif world > 1:      # gloo control plane (--share-gpu): reduce on the host
        msc, nlc = ms.cpu(), nl.cpu()
        dist.all_reduce(msc, op=dist.ReduceOp.MAX)
        dist.all_reduce(nlc, op=dist.ReduceOp.SUM)
        ms, nl = msc, nlc
    ms = float(ms.item())
    diag = slab.combine_diagnostics(plan.diagnostics(a), rank, world)   # whole domain, rank order
    if diag["nonfinite"]:
        raise SystemExit(f"bench: populations diverged ({wl.name})")
    cells_rank = nx * ny * nzl
    out = {"value": cells_rank * world * steps / (ms * 1e-3) / 1e6, "ms": ms,
           "launches": int(nl.item()), "transport": transport, "kernel": kernel_name,
           "cells_rank": cells_rank, "diag": diag,
           "clocks": sampler.summary() if sampler else None,
           "host_us_per_step": (runner.host_us_per_step if runner is not None
                                and runner.host_us_per_step is not None
                                else host_enqueue / steps * 1e6),
           "host_loop": ("mlb_slab_run_steps (one library call for the whole loop)"
                         if runner is not None and runner.ring is not None and runner.c_loop
                         else "per-step Python schedule" if runner is not None
                         else "mlb_run_steps (one library call)")}
    if runner is not None and runner.ring is not None:
        runner.ring.close()
    del a, b, runner
    plan.close()
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.preflight_child:
        return preflight_child(args)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    prec_tok = args.precision

    if args.impl == "reference":
        if rank != 0:
            return 0
        wl = Workload("default", max(1, args.gpus), args.n, args.scaling)
        n = wl.nx
        base, ms = cpu_arm(n, prec_tok, args.steps, args.warmup, budget_s=120.0)
        line = {
            "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "MLUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": PREC_DTYPE[prec_tok], "data": "synthetic",
            "config": wl.describe(prec_tok),
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "MLUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
        }
        print(json.dumps(line), flush=True)
        return 0

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2409_16781_b200 import _cabi, cases, engine, slab
    from paper_2409_16781_b200.fields import Layout, Precision
    from paper_2409_16781_b200.kernels import KernelPlan, pinned_empty

    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run "
                             "(one rank per GPU)")
    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    fdev = None if args.share_gpu else device    # device of control-plane tensors (None: host)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    prec = Precision.from_token(prec_tok)
    itemsize = prec.storage.itemsize
    wl = Workload(args.config, world, args.n, args.scaling, args.inplace)
    slab_mode = world > 1 or args.force_slab

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- N > 1: bitwise preflight through the runners that get timed ---------
    # In a child process per rank with a time limit.  If the fused peer-store exchange
    # fails it (mismatch, error or no answer) the run falls back to the send/recv
    # transport - preflighted the same way - and says so; if that fails too the bench
    # aborts: a number from a path that does not reproduce the oracle is worthless.
    pre = None
    if slab_mode and not args.no_preflight:
        def agreed(rec):
            ok = torch.tensor([1 if rec.get("result") == "bitwise" else 0], dtype=torch.int32,
                              device=device if (world > 1 and fdev is not None) else "cpu")
            if world > 1:
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            return bool(ok.item())
        pre = preflight_guarded(args, world)
        if not agreed(pre) and args.transport == "peer":
            first = pre.get("result", "?")
            args.transport = "nccl"
            pre = preflight_guarded(args, world)
            pre["fallback"] = f"the peer-memory ring failed the preflight on some rank ({first}); " \
                              f"halo exchange by send/recv instead"
        if not agreed(pre):
            raise SystemExit(f"bench preflight failed: {pre.get('result')}")

    # ---- device-timed run: W warm-up, then exactly K steps -------------------
    main_run = run_device(wl, args, prec_tok, rank, world, device, fdev, args.steps, args.warmup,
                          clocks=rank == 0)
    ms, value = main_run["ms"], main_run["value"]
    cells_rank = main_run["cells_rank"]

    # ---- end to end through the host API ------------------------------------
    e2e = None
    state = None
    if not args.no_e2e and not (wl.name == "c3-strong" and world == 1):
        h2d = 19 * cells_rank * itemsize + cells_rank      # populations + flags
        d2h = 19 * cells_rank * itemsize
        if not slab_mode:
            # the public call: a host state as the reference's driver holds it
            vals = wl.init_values(prec.storage)
            data = pinned_empty((19, cells_rank), prec.storage)
            for q in range(19):
                data[q].fill(vals[q])
            from paper_2409_16781_b200.fields import PopulationField
            from paper_2409_16781_b200.lattice import RelaxationParams
            mask = pinned_empty((cells_rank,), np.uint8)   # page-locked, as cases.init makes it
            np.copyto(mask.reshape(wl.nz, wl.ny, wl.nx), wl.planes(0, wl.nz))
            state = engine.SimState(
                f_pre=PopulationField(data, wl.nx, wl.ny, wl.nz, Layout.ROW), f_post_=None,
                mask=mask, nx=wl.nx, ny=wl.ny, nz=wl.nz,
                layout=Layout.ROW, precision=prec, params=RelaxationParams.from_omega(wl.omega),
                wall_u=wl.wall_u, inlet_u=wl.inlet_u, case=wl.case)
            cfg = engine.RunConfig(steps=args.steps, precision=prec, device=local,
                                   inplace=wl.inplace)
            warm = engine.RunConfig(steps=max(1, args.warmup), precision=prec, device=local,
                                    inplace=wl.inplace)
            engine.run(state, warm)              # allocator / page-lock warm-up, untimed
            barrier()
            t0 = time.perf_counter()
            engine.run(state, cfg)               # H2D + K steps + D2H
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        else:
            z0 = rank * wl.nzl
            flags = wl.planes(z0, z0 + wl.nzl)
            lo, hi = wl.planes(z0 - 1, z0)[0], wl.planes(z0 + wl.nzl, z0 + wl.nzl + 1)[0]
            vals = wl.init_values(prec.storage)
            host = pinned_empty((19, cells_rank), prec.storage)
            for q in range(19):
                host[q].fill(vals[q])

            def e2e_once(k):
                p = KernelPlan(wl.nx, wl.ny, wl.nzl, Layout.ROW, prec, flags, wl.omega, wl.wall_u,
                               inlet_u=wl.inlet_u, device=local, halo_lo=lo, halo_hi=hi, slab=True)
                x = p.alloc()
                p.upload(host, x)
                if wl.inplace:
                    rr = slab.open_inplace_runner(p, x, rank, world)
                    rr.c_loop = not args.python_loop
                    rr.run_inplace(x, k)
                    rr.normalize(x)
                else:
                    y = p.alloc()
                    y.tensor.copy_(x.tensor)
                    try:
                        p.set_passthrough(True)
                    except ValueError:
                        p.set_passthrough(False)
                    rr, _ = slab.open_runner(p, x, y, rank, world, transport=args.transport)
                    rr.c_loop = not args.python_loop
                    x, y = rr.run(x, y, k)
                    rr.finish()
                p.download(x, host)
                if rr.ring is not None:
                    rr.ring.close()
                p.close()
            e2e_once(max(1, args.warmup))
            barrier()
            t0 = time.perf_counter()
            e2e_once(args.steps)
            barrier()
            dt = time.perf_counter() - t0
        dtt = torch.tensor([dt], dtype=torch.float64)
        if world > 1:
            if fdev is not None:
                dtt = dtt.to(device)
            dist.all_reduce(dtt, op=dist.ReduceOp.MAX)
        dt = float(dtt.item())
        e2e = {"value": cells_rank * world * args.steps / dt / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": h2d * world / args.steps,
               "d2h_bytes_per_step": d2h * world / args.steps,
               "seconds": dt,
               "call": "engine.run(host state, RunConfig(steps=K)): upload, K steps, download"
                       if not slab_mode else
                       "per rank: KernelPlan + upload, halo transport setup, DistSlab.run(K), download"}

    # ---- N = 1: the timed configuration against the oracle, full size ---------
    parity, cpu_base = None, None
    if world == 1 and not slab_mode and not args.no_cpu_baseline and state is not None:
        psteps = 4
        try:
            vals = wl.init_values(prec.storage)
            f_init = np.empty((19, cells_rank), dtype=prec.storage)
            for q in range(19):
                f_init[q].fill(vals[q])

            def gpu_after(k):
                # the benchmark's own initial state, k steps through the timed path
                for q in range(19):
                    state.f_pre.data[q].fill(vals[q])
                state.t = 0
                engine.run(state, engine.RunConfig(steps=k, precision=prec, device=local,
                                                   inplace=wl.inplace))
                return state.f_pre.data
            parity, cpu_base = parity_and_cpu_baseline(wl, prec_tok, state.mask, f_init, gpu_after,
                                                       psteps)
        except MemoryError as exc:
            parity = {"result": "skipped", "why": f"host memory: {exc}"}
        if parity.get("result") == "MISMATCH":
            print(json.dumps({"error": "bench: GPU populations differ from the CPU oracle",
                              "parity": parity}), flush=True)
            return 1
    elif world == 1 and not args.no_cpu_baseline:
        cpu_base, _ = cpu_arm(wl.nx, prec_tok, steps=10, warmup=2, budget_s=15.0)
    state = None

    # ---- the other BASELINE configurations, briefly ---------------------------
    extra = None
    want_extra = (world == 1 and not args.no_extra and args.config == "default"
                  and not args.n and prec_tok == "single" and not slab_mode) \
        or (world > 1 and args.extra)
    if want_extra:
        extra = {}

        def on_alarm(signum, frame):
            raise TimeoutError("extra workloads timed out")
        signal.signal(signal.SIGALRM, on_alarm)
        todo = [("c3-strong", "single", 20), ("c3-weak", "single", 20), ("c4", "single", 20)]
        if world == 1:
            todo += [("c0", "double", 100), ("c1", "double", 50), ("c1", "single", 50)]
        for name, xprec, xsteps in todo:
            if world == 1 and name == "c3-weak":
                continue        # 1024 x 1024 x 128 on one GPU says nothing c3-strong does not
            key = name if name not in ("c0", "c1") else f"{name}-{PREC_TAG[xprec]}"
            try:
                signal.alarm(300)
                xw = Workload(name, world)
                # (c0 replays its loop from a CUDA graph: captured during the warm-up)
                xwarm = 64 if name == "c0" else 3
                r = run_device(xw, args, xprec, rank, world, device, fdev, xsteps, xwarm)
                signal.alarm(0)
                extra[key] = {
                    "workload": xw.describe(xprec, r["transport"])["workload"],
                    "l2_policy": xw.describe(xprec)["l2_policy"],
                    "value": r["value"], "unit": "MLUPS", "steps": xsteps, "warmup": xwarm,
                    "bytes_per_update": 38 * PREC_BYTES[xprec],
                    "ms_per_step": r["ms"] / xsteps, "blocks_per_gpu": 1 if xw.inplace else 2,
                    "nz_per_gpu": xw.nzl, "cells_per_gpu": r["cells_rank"], "kernel": r["kernel"],
                    "frac_of_hbm_peak": None, "host_us_per_step": r["host_us_per_step"],
                    "check": {"mass": r["diag"]["mass"], "max_u": r["diag"]["max_u"]}}
            except (Exception, SystemExit) as exc:   # never lose the main line to an extra
                signal.alarm(0)
                extra[key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
                if world > 1:
                    break       # the ranks may no longer be in step

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the fused kernel ---------------------------------------
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak, peak_src = json.load(open(peaks_path))["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    bytes_per_update = 2 * 19 * itemsize
    kernel_ms = ms / args.steps           # one fused-kernel launch per step per GPU
    achieved = bytes_per_update * cells_rank / (kernel_ms * 1e-3) / 1e9
    traffic, traffic_note = None, "no ncu record for this kernel / size in profiles/traffic.json"
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and wl.nx == wl.ny == wl.nzl:
        table = json.load(open(tpath))
        tag, n = PREC_TAG[prec_tok], wl.nx
        keys = ([f"aa_pull_{tag}_{n}", f"aa_local_{tag}_{n}"] if wl.inplace
                else [f"step_kernel_{tag}_{n}"])
        recs = [table.get(k) for k in keys]
        if all(isinstance(r, dict) for r in recs):
            build = _cabi.build_id()
            if all(r.get("build_id") == build for r in recs):
                traffic = sum(r["bytes"] for r in recs) / len(recs)   # per launch (halves alternate)
                traffic_note = f"ncu dram__bytes_read.sum + dram__bytes_write.sum, build {build}"
            else:
                traffic_note = (f"profiles/traffic.json was recorded for build "
                                f"{recs[0].get('build_id')}, this library is build {build}: "
                                f"re-run tools/profile_round.sh")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note,
                "peak_source": peak_src,
                "kernel": main_run["kernel"], "algorithmic_bytes_per_update": bytes_per_update,
                "updates_per_launch": cells_rank, "kernel_ms": kernel_ms}
    if extra:
        for name, rec in extra.items():
            if "ms_per_step" in rec:
                rec["frac_of_hbm_peak"] = (rec["bytes_per_update"] * rec["cells_per_gpu"]
                                           / (rec["ms_per_step"] * 1e-3) / 1e9 / peak)

    ref2d = None
    if world == 1 and not args.no_cpu_baseline:
        ref2d = ref2d_arm()

    config = wl.describe(prec_tok, main_run["transport"])
    if main_run["transport"]:
        config["signal_wait"] = {1: "stream memory operation", 2: "polling kernel"}[
            _cabi.lib().mlb_signal_wait_kind()]
    if pre is not None:
        config["preflight_parity"] = pre["result"]
    host = {"loop": main_run["host_loop"], "us_per_step": main_run["host_us_per_step"]}
    diag = main_run["diag"]
    line = {
        "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if wl.strong and world > 1 else "weak",
        "vs_baseline": None,
        "dtype": PREC_DTYPE[prec_tok], "data": "synthetic",
        "config": config,
        "clocks": main_run["clocks"], "e2e": e2e, "gpu_launches": main_run["launches"],
        "roofline": roofline, "cpu_baseline": cpu_base, "parity": parity,
        "cpu_baseline_ref2d": ref2d, "extra": extra, "preflight": pre, "host": host,
        "build_id": _cabi.build_id(),
        "check": {"mass": diag["mass"], "max_u": diag["max_u"], "nonfinite": diag["nonfinite"]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
