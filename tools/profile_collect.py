"""Turn the captures of tools/profile_round.sh (gpurun_out/) into the tracked
summaries under profiles/."""
import csv, collections, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"

def shares(src, dst, title):
    rows = [r for r in csv.reader(open(src)) if r and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        k = r[4]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r[-1]) / 1e6)
    total = sum(t for _, t in agg.values())
    with open(dst, "w") as fh:
        fh.write(f"# {title}\n# per-launch times are cold-cache and serialised: compare SHARES, not absolutes\n")
        fh.write("kernel,launches,total_ms,share_of_captured,avg_ms\n")
        for k, (n, t) in agg.items():
            fh.write(f"\"{k}\",{n},{t:.3f},{t / total:.4f},{t / n:.4f}\n")

import shutil
shutil.copy(os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, f"launches_bench_{tag}.csv"))
shares(os.path.join(OUT, "launches_bench.csv"), os.path.join(PROF, f"launch_shares_{tag}.csv"),
       "ncu launch list of `python bench.py --steps 10 --warmup 3 --no-cpu-baseline`")
if os.path.exists(os.path.join(OUT, "launches_slab.csv")):
    shares(os.path.join(OUT, "launches_slab.csv"), os.path.join(PROF, f"launch_shares_slab_{tag}.csv"),
           "ncu launch list of `python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-slab` "
           "(z-slab driver, fused peer-store exchange, world 1)")
traffic = {}
for name, key in (("step_f32_512", "step_kernel_f32_512"), ("step_f64_512", "step_kernel_f64_512"),
                  ("step_f16_512", "step_kernel_f16_512"), ("aa_pull_f32_512", "aa_pull_f32_512"),
                  ("aa_local_f32_512", "aa_local_f32_512")):
    summary = os.path.join(OUT, f"ncu_{name}.txt")
    if not os.path.exists(summary):
        continue
    txt = open(summary).read()
    open(os.path.join(PROF, f"ncu_{name}_{tag}.txt"), "w").write(txt)
    rd = wr = None
    for ln in txt.splitlines():
        p = ln.split()
        if "dram__bytes_read.sum" in ln: rd = float(p[1]) * {"Gbyte": 1e9, "Mbyte": 1e6}[p[2]]
        if "dram__bytes_write.sum" in ln: wr = float(p[1]) * {"Gbyte": 1e9, "Mbyte": 1e6}[p[2]]
    if rd and wr:
        traffic[key] = rd + wr
json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
