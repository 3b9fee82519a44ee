"""Throughput, arithmetic intensity and roofline metrics for the D3Q19 loop.

Mirror of the measurement definitions in
/root/reference/pkg/src/lb2d/perfport.py (`FLOPS_PER_CELL` :16-27,
`bytes_per_cell` :40-45, `arithmetic_intensity` :48-52, `mlups` :55-61,
`roofline_peak` :64-72, `roofline_efficiency` :75-81), restated for 19
velocities.  The update-rate currency is MLUPS: million lattice-site
updates per second, ALL grid cells (solid included) times steps over
update-loop seconds.  The cost model is per fused cell update and assumes
the pull kernel's ideal traffic - each population plane read once and
written once; flag traffic is not modelled, exactly as in the reference
(perfport.py:5-7) - it feeds the roofline estimate, not the timer.

The reference's cross-vendor portability analytics (`pp_metric`,
`estimate_cross_platform_flop_rate`, `expand_axes`) are out of scope.
"""

from .fields import Precision
from .lattice import Q

#: Arithmetic cost of one fused cell update, counted on the canonical
#: per-cell expression (lattice.collide_cell) by the reference's rule
#: (adds/subs + muls + divs):
#:
#:   moments (rho, momentum, 1/rho, u)            49
#:   speed-square and common factor (1 - 1.5u^2)   7
#:   equilibrium, nine opposite pairs sharing     82
#:   BGK relaxation, 19 directions x 3            57
#:   total                                       195
#:
#: Re-derived in tests/test_lattice.py by replaying the expression with
#: operation-counting numbers.
FLOPS_PER_CELL = 195


def flops_per_cell(precision=None):
    return FLOPS_PER_CELL


def bytes_per_cell(precision):
    """Ideal memory traffic per cell update: 19 planes read + 19 written in
    storage precision (152 B in fp32, 304 B in fp64, 76 B in mixed1)."""
    if not isinstance(precision, Precision):
        precision = Precision.from_token(precision)
    return 2 * Q * precision.storage.itemsize


def arithmetic_intensity(flops, nbytes):
    if nbytes <= 0:
        raise ValueError("byte count must be positive")
    return flops / nbytes


def mlups(nx, ny, nz, steps, seconds):
    """Million lattice-site updates per second."""
    if seconds <= 0.0:
        raise ValueError("elapsed seconds must be positive")
    if nx < 1 or ny < 1 or nz < 1 or steps < 1:
        raise ValueError("grid sizes and steps must be positive")
    return nx * ny * nz * steps / (seconds * 1e6)


def roofline_peak(fr_peak, bandwidth, ai):
    """Attainable rate under the roofline: min(FR, BW * AI)."""
    if fr_peak <= 0 or bandwidth <= 0 or ai <= 0:
        raise ValueError("roofline inputs must be positive")
    return min(fr_peak, bandwidth * ai)


def roofline_efficiency(achieved, peak):
    if peak <= 0:
        raise ValueError("peak rate must be positive")
    if achieved < 0:
        raise ValueError("achieved rate cannot be negative")
    return achieved / peak


def achieved_bandwidth_gbs(mlups_value, precision):
    """Algorithmic GB/s implied by an update rate: MLUPS x bytes per update."""
    return mlups_value * 1e6 * bytes_per_cell(precision) / 1e9


def bandwidth_ceiling_mlups(bandwidth_gbs, precision):
    """The update rate at which the ideal traffic saturates `bandwidth_gbs`."""
    return bandwidth_gbs * 1e9 / bytes_per_cell(precision) / 1e6


# --------------------------------------------------------------------------
# The reference's sweep protocol (perfport.py:156-184) on the CUDA path.
class PerfRecord:
    """Outcome of one benchmark job (fields follow lb2d's PerfRecord, plus the
    third dimension and the bandwidth view this path is judged by)."""

    FIELDS = ("case", "nx", "ny", "nz", "precision", "layout", "schedule", "inplace", "steps",
              "seconds", "mlups", "flops_per_cell", "bytes_per_cell", "ai", "gbs", "error")

    def __init__(self, spec, config):
        nbytes = bytes_per_cell(config.precision)
        self.case, self.nx, self.ny, self.nz = spec.name, spec.nx, spec.ny, spec.nz
        self.precision = config.precision.token
        self.layout = config.layout.token
        self.schedule = config.schedule.label()
        self.inplace = bool(config.inplace)
        self.steps = config.steps
        self.seconds = self.mlups = self.gbs = 0.0
        self.flops_per_cell = FLOPS_PER_CELL
        self.bytes_per_cell = nbytes
        self.ai = arithmetic_intensity(FLOPS_PER_CELL, nbytes)
        self.error = ""

    def as_dict(self):
        return {k: getattr(self, k) for k in self.FIELDS}

    def __repr__(self):
        return f"PerfRecord({self.as_dict()})"


def bench_sweep(jobs, reps=3, progress=None):
    """Time (CaseSpec, RunConfig) jobs the way the reference does: one
    discarded warm-up run, then `reps` runs each from a freshly initialised
    state; the record carries the MEDIAN update-loop time (device time, CUDA
    events - `RunStats.seconds`).  A job that raises is recorded with its
    error and the sweep goes on."""
    import statistics

    from . import cases, engine  # deferred: metric-only users never touch the GPU path

    if reps < 1:
        raise ValueError("reps must be >= 1")
    out = []
    for spec, config in jobs:
        rec = PerfRecord(spec, config)
        try:
            samples = []
            for attempt in range(reps + 1):          # attempt 0 is the warm-up
                state = cases.init(spec, config.precision, config.layout)
                seconds = engine.run(state, config).seconds
                if attempt:
                    samples.append(seconds)
            rec.seconds = statistics.median(samples)
            rec.mlups = mlups(spec.nx, spec.ny, spec.nz, config.steps, rec.seconds)
            rec.gbs = achieved_bandwidth_gbs(rec.mlups, config.precision)
        except Exception as exc:  # noqa: BLE001 - one bad job must not end the sweep
            rec.error = f"{type(exc).__name__}: {exc}"
        out.append(rec)
        if progress is not None:
            progress(rec)
    return out
