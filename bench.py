#!/usr/bin/env python
"""bench.py - MLUPS of the D3Q19 BGK time-step loop on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[2], the one the metric is quoted on):
D3Q19 BGK lid-driven cavity, 512^3 cells per GPU, fp32, Re 1000, u0 0.1.
With N > 1 (launched under torch.distributed.run, one rank per GPU) the
cavity is 512 x 512 x (512 N), split into N z-slabs with 5-population halo
exchange over NCCL - per-GPU work is fixed, i.e. weak scaling.

One "step" is one lattice time step: the fused pull-stream + BGK collide
kernel over all cells (plus the open-boundary pass, a no-op for the cavity,
and the halo exchange when N > 1).  MLUPS counts ALL cells, solid included,
like the reference (lb2d perfport.py:55-61, engine.py:270-271).

The one JSON line carries
  value      device-timed whole-job MLUPS, populations resident in HBM;
             CUDA events on the launching stream, max over ranks;
  e2e        the same K steps through the public host API
             (`engine.run` on a host-resident state in pinned memory):
             H2D of the populations + flags, K steps, D2H of the result,
             all inside the timed region;
  roofline   the fused kernel against the measured HBM bandwidth
             (MEASURED_PEAKS.json): algorithmic bytes 2 x 19 x 4 B per
             update (lb2d perfport.py:40-45 with Q = 19);
  cpu_baseline  the CPU oracle (a port of the reference's algorithm,
             OpenMP, all host cores) on a bounded sample of the workload.

`--impl reference` times that CPU port alone, on the same config, each step
a bounded z-slice of the cavity so the run ends within a few minutes.  The
oracle is used here as the measured CPU arm only; it is never on the GPU
path.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX = NY = NZ_PER_GPU = 512
RE, U0 = 1000.0, 0.1
METRIC = "MLUPS (D3Q19 BGK)"
PREC_NAME = {"single": "fp32", "double": "fp64", "mixed1": "fp16 storage / fp32 compute",
             "mixed2": "fp32 storage / fp64 compute"}
PREC_BYTES = {"single": 4, "double": 8, "mixed1": 2, "mixed2": 4}
PREC_DTYPE = {"single": "f32", "double": "f64", "mixed1": "f16 storage, f32 compute",
              "mixed2": "f32 storage, f64 compute"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--edge", "--n", dest="n", type=int, default=0,
                    help="override the edge length (debug; use --edge under torchrun)")
    ap.add_argument("--precision", default="single", choices=["single", "double", "mixed1", "mixed2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-slab", action="store_true",
                    help="run the z-slab driver (halo planes, boundary-first overlap) even on 1 GPU")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="halo exchange of the z-slab run: 'peer' = stores into the neighbours' halo "
                         "planes from inside the fused kernel over CUDA-IPC-mapped peer memory "
                         "(default; falls back to 'nccl' if the mapping cannot be set up), "
                         "'nccl' = torch.distributed send/recv")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: 'weak' = 512^3 cells per GPU (default, what the driver's scaling run "
                         "measures), 'strong' = the N = 1 domain (512^3) split into N z-slabs")
    ap.add_argument("--inplace", action="store_true",
                    help="the in-place update (one population block per GPU instead of two; same "
                         "arithmetic and traffic)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="debug, not a benchmark: all ranks use device 0 with a gloo control plane, so "
                         "a one-GPU box can drive the N > 1 code path (peer ring across processes)")
    ap.add_argument("--variant", type=int, default=0, help="kernel variant (tuning; see mlb_plan_set_variant)")
    return ap.parse_args()


def workload_config(n, nz_global, world, prec, omega, inplace=False, strong=False):
    size = f"{n}^3" if nz_global == n else f"{n}x{n}x{nz_global}"
    return {
        "workload": f"D3Q19 BGK lid-driven cavity {size} {PREC_NAME[prec]}"
                    f" (BASELINE.json configs[2]"
                    f"{', z-slab ' + ('strong' if strong else 'weak') + ' scaling' if world > 1 else ''})",
        "nx": n, "ny": n, "nz_per_gpu": nz_global // world, "nz_global": nz_global,
        "re": RE, "u0": U0, "omega": omega,
        "decomposition": f"{world} z-slab(s), 5-population halos" if world > 1 else "single GPU",
        "blocks_per_gpu": 1 if inplace else 2,
        "l2_policy": f"inputs exceed L2: {'one population block' if inplace else 'two population blocks'} of "
                     f"{19 * n * n * (nz_global // world) * PREC_BYTES[prec] / 1e9:.1f} GB per GPU vs 126 MB L2",
    }


# --------------------------------------------------------------------------
# clocks: sample nvidia-smi during the timed region (B200_PROFILING.md)
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

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
        for r in self.rows:
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
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


# --------------------------------------------------------------------------
def slab_mask(n, nzl, rank, world):
    """This rank's [x, y, z] flag block (nzl planes) of the cavity that the ranks'
    slabs stack up to."""
    import numpy as np
    from paper_2409_16781_b200 import boundaries as B
    m = B.cavity_mask(n, n, nzl, z_walls=False)
    if rank == 0:
        m[:, :, 0] = B.SOLID
    if rank == world - 1:
        m[:, :, -1] = B.SOLID
    return np.ascontiguousarray(m)


def cpu_arm(n, prec, steps, warmup, budget_s):
    """Time the CPU port of the reference algorithm (the oracle, OpenMP over
    all host cores) on a bounded z-slice of the cavity."""
    import numpy as np
    from oracle.cpu import CpuOracle
    from paper_2409_16781_b200 import boundaries as B
    from paper_2409_16781_b200.lattice import W, omega_from_reynolds
    cores = os.cpu_count() or 1
    dtype = {"single": np.float32, "double": np.float64, "mixed1": np.float16,
             "mixed2": np.float32}[prec]
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


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n = args.n or NX
    prec_tok = args.precision

    if args.impl == "reference":
        if rank != 0:
            return 0
        from paper_2409_16781_b200.lattice import omega_from_reynolds
        omega = omega_from_reynolds(RE, U0, n).omega
        base, ms = cpu_arm(n, prec_tok, args.steps, args.warmup, budget_s=120.0)
        line = {
            "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "MLUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": PREC_DTYPE[prec_tok], "data": "synthetic",
            "config": workload_config(n, n * max(1, args.gpus), max(1, args.gpus), prec_tok, omega),
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
    from paper_2409_16781_b200 import _cabi, boundaries as B, cases, engine, slab
    from paper_2409_16781_b200.fields import Layout, Precision
    from paper_2409_16781_b200.kernels import KernelPlan, pinned_empty
    from paper_2409_16781_b200.lattice import W, omega_from_reynolds

    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run "
                             "(one rank per GPU)")
    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    prec = Precision.from_token(prec_tok)
    itemsize = prec.storage.itemsize
    strong = args.scaling == "strong" and world > 1
    if strong and n % world:
        raise SystemExit(f"--scaling strong needs {n} planes to split evenly over {world} ranks")
    nzl = n // world if strong else n              # planes per rank
    nz_global = nzl * world
    params = omega_from_reynolds(RE, U0, n)
    cells_rank = n * n * nzl
    cells_all = cells_rank * world

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- host state (pinned) and the plan ----------------------------------
    slab_mode = world > 1 or args.force_slab
    if not slab_mode:
        spec = cases.CaseSpec("ldc", n, n, n, re=RE, u0=U0)
        state = cases.init(spec, prec)
        mask_flat = state.mask
        plan = KernelPlan(n, n, n, Layout.ROW, prec, mask_flat, params.omega,
                          (U0, 0.0, 0.0), device=local)
        host = state.f_pre.data
    else:
        m = slab_mask(n, nzl, rank, world)
        mask_flat = B.flatten_mask(m)
        lo, hi = slab.exchange_flag_halos(mask_flat.reshape(nzl, n, n), rank, world,
                                          device=None if args.share_gpu else device)
        plan = KernelPlan(n, n, nzl, Layout.ROW, prec, mask_flat, params.omega,
                          (U0, 0.0, 0.0), device=local, halo_lo=lo, halo_hi=hi, slab=True)
        host = pinned_empty((19, cells_rank), prec.storage)
        for q in range(19):
            host[q].fill(W[q])
    if args.variant:
        plan.set_variant(args.variant)
    kernel_name = plan.kernel_name if not args.inplace else \
        "mlb::aa_pull_vec_kernel + mlb::aa_local_vec_kernel (alternating)"
    a = plan.alloc()
    plan.upload(host, a)
    runner = None
    transport = None
    if args.inplace:
        b = None
        if slab_mode:
            runner, transport = slab.open_inplace_runner(plan, a, rank, world), "peer"
    else:
        b = plan.alloc()
        b.tensor.copy_(a.tensor)
        plan.set_passthrough(True)   # both blocks identical: what engine.Session establishes

    def make_runner(p, x, y):
        return slab.open_runner(p, x, y, rank, world, transport=args.transport)

    if slab_mode and not args.inplace:
        runner, transport = make_runner(plan, a, b)

    def advance(x, y, k):
        if args.inplace:
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
        if runner is not None and args.inplace:
            runner.normalize(x)
        elif runner is not None:
            runner.finish()
        elif args.inplace:
            plan.normalize(x)

    # ---- device-timed run: W warm-up, then exactly K steps -------------------
    a, b = advance(a, b, args.warmup)
    if not args.inplace:
        settle(a)
    elif runner is not None:
        runner.finish()
    barrier()
    if runner is not None and runner.ring is not None and not args.inplace:
        # the fused exchange against the plain one, on live data: the halos the
        # kernels stored into this rank must be the planes send/recv delivers
        if not slab.halos_match_send_recv(plan, a, rank, world):
            raise SystemExit("bench: fused peer-store halos differ from the send/recv exchange")
    launches0 = _cabi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        a, b = advance(a, b, args.steps)
        e1.record()
        if runner is not None:
            runner.finish()
        barrier()
    settle(a)
    launches = _cabi.launch_count() - launches0
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    nl = torch.tensor([launches], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    ms = float(ms.item())
    value = cells_all * args.steps / (ms * 1e-3) / 1e6
    diag = slab.combine_diagnostics(plan.diagnostics(a), rank, world)   # whole domain, rank order
    if diag["nonfinite"]:
        raise SystemExit("bench: populations diverged")

    # ---- end to end through the host API ------------------------------------
    e2e = None
    if not args.no_e2e:
        h2d = 19 * cells_rank * itemsize + cells_rank      # populations + flags
        d2h = 19 * cells_rank * itemsize
        if runner is not None and runner.ring is not None:
            runner.ring.close()
        del a, b, runner
        plan.close()
        torch.cuda.empty_cache()
        if not slab_mode:
            cfg = engine.RunConfig(steps=args.steps, precision=prec, device=local,
                                   inplace=args.inplace)
            warm = engine.RunConfig(steps=max(1, args.warmup), precision=prec, device=local,
                                    inplace=args.inplace)
            engine.run(state, warm)              # allocator / page-lock warm-up, untimed
            barrier()
            t0 = time.perf_counter()
            engine.run(state, cfg)               # H2D + K steps + D2H
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        else:
            def e2e_once(k):
                p = KernelPlan(n, n, nzl, Layout.ROW, prec, mask_flat, params.omega,
                               (U0, 0.0, 0.0), device=local, halo_lo=lo, halo_hi=hi, slab=True)
                x = p.alloc()
                p.upload(host, x)
                if args.inplace:
                    rr = slab.open_inplace_runner(p, x, rank, world)
                    rr.run_inplace(x, k)
                    rr.normalize(x)
                else:
                    y = p.alloc()
                    y.tensor.copy_(x.tensor)
                    p.set_passthrough(True)
                    rr, _ = make_runner(p, x, y)
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
        dtt = torch.tensor([dt], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(dtt, op=dist.ReduceOp.MAX)
        dt = float(dtt.item())
        e2e = {"value": cells_all * args.steps / dt / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": h2d * world / args.steps,
               "d2h_bytes_per_step": d2h * world / args.steps,
               "seconds": dt,
               "call": "engine.run(host state, RunConfig(steps=K)): upload, K steps, download"
                       if not slab_mode else
                       "per rank: KernelPlan + upload, halo transport setup, DistSlab.run(K), download"}


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
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        key = f"step_kernel_{ {'single': 'f32', 'double': 'f64', 'mixed1': 'f16', 'mixed2': 'm2'}[prec_tok] }_{n}"
        table = json.load(open(tpath))
        traffic = table.get(key)
        if args.inplace:   # the two halves alternate: per-launch average
            tag = {'single': 'f32', 'double': 'f64', 'mixed1': 'f16', 'mixed2': 'm2'}[prec_tok]
            pair = [table.get(f"aa_pull_{tag}_{n}"), table.get(f"aa_local_{tag}_{n}")]
            traffic = sum(pair) / 2 if all(pair) else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "kernel": kernel_name, "algorithmic_bytes_per_update": bytes_per_update,
                "updates_per_launch": cells_rank, "kernel_ms": kernel_ms}

    cpu_base = None
    if world == 1 and not args.no_cpu_baseline:
        cpu_base, _ = cpu_arm(n, prec_tok, steps=10, warmup=2, budget_s=15.0)

    line = {
        "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": PREC_DTYPE[prec_tok], "data": "synthetic",
        "config": dict(workload_config(n, nz_global, world, prec_tok, params.omega, args.inplace,
                                       strong),
                       **({"halo_transport": transport,
                           "signal_wait": {1: "stream memory operation", 2: "polling kernel"}[
                               _cabi.lib().mlb_signal_wait_kind()]} if transport else {})),
        "clocks": clk.summary(), "e2e": e2e, "gpu_launches": int(nl.item()),
        "roofline": roofline, "cpu_baseline": cpu_base,
        "check": {"mass": diag["mass"], "max_u": diag["max_u"], "nonfinite": diag["nonfinite"]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
