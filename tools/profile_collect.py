"""Turn the captures of tools/profile_round.sh (gpurun_out/) into the tracked
summaries under profiles/.  profiles/traffic.json records, per kernel, the ncu
DRAM byte count TOGETHER WITH the build id of the library that was profiled
(mlb_build_id(): hash of the sources); bench.py quotes a figure only for the
build it belongs to."""
import csv, collections, json, os, shutil, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
build = open(os.path.join(OUT, "build_id.txt")).read().strip()

def shares(src, dst, title):
    rows = [r for r in csv.reader(open(src)) if r and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        k = r[4]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r[-1]) / 1e6)
    total = sum(t for _, t in agg.values())
    with open(dst, "w") as fh:
        fh.write(f"# {title}\n# library build {build}\n"
                 f"# per-launch times are cold-cache and serialised: compare SHARES, not absolutes\n")
        fh.write("kernel,launches,total_ms,share_of_captured,avg_ms\n")
        for k, (n, t) in agg.items():
            fh.write(f"\"{k}\",{n},{t:.3f},{t / total:.4f},{t / n:.4f}\n")

shutil.copy(os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, f"launches_bench_{tag}.csv"))
shares(os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, f"launch_shares_{tag}.csv"),
       "ncu launch list of `python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra`")
if os.path.exists(os.path.join(OUT, "launches_slab.csv")):
    shares(os.path.join(OUT, "launches_slab.csv"), os.path.join(PROF, f"launch_shares_slab_{tag}.csv"),
           "ncu launch list of `python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-slab "
           "--no-preflight` (z-slab driver, fused peer-store exchange, one-call loop, world 1)")
traffic = {}
names = [(f"{k}_{t}_512", f"{'step_kernel' if k == 'step' else k}_{t}_512")
         for t in ("f32", "f64", "f16", "m2") for k in ("step", "aa_pull", "aa_local")]
names += [("stage_f16_512", "stage_f16_512"), ("aa_pull_rowb_f32_512", "aa_pull_rowb_f32_512")]
names += [(f"diag_{t}_512", f"diag_{t}_512") for t in ("f32", "f64", "f16")]
for name, key in names:
    summary = os.path.join(OUT, f"ncu_{name}.txt")
    if not os.path.exists(summary):
        continue
    txt = open(summary).read()
    open(os.path.join(PROF, f"ncu_{name}_{tag}.txt"), "w").write(f"# library build {build}\n" + txt)
    rd = wr = ms = None
    for ln in txt.splitlines():
        p = ln.split()
        if "dram__bytes_read.sum" in ln: rd = float(p[1]) * {"Gbyte": 1e9, "Mbyte": 1e6}[p[2]]
        if "dram__bytes_write.sum" in ln: wr = float(p[1]) * {"Gbyte": 1e9, "Mbyte": 1e6}[p[2]]
        if "gpu__time_duration.sum" in ln: ms = float(p[1]) * {"ms": 1.0, "us": 1e-3}.get(p[2], 1.0)
    if rd and wr:
        traffic[key] = {"bytes": rd + wr, "build_id": build, "ncu_ms": ms,
                        "source": f"profiles/ncu_{name}_{tag}.txt"}
json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
