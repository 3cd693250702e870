"""Write the per-round profile summaries under profiles/:
  python tools/make_profiles.py r02 gpurun_out/launches_r02.csv gpurun_out/prof_r02b.ncu-rep"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

tag, launches = sys.argv[1:3]
reps = sys.argv[3:]
os.makedirs("profiles", exist_ok=True)
rows = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.OrderedDict()
for r in data:
    if len(r) < len(hdr) or r[mn] != "gpu__time_duration.sum":
        continue
    a = agg.setdefault(r[kn].split("(")[0], [0, 0.0])
    a[0] += 1
    a[1] += float(r[mv].replace(",", ""))
lines = [f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none -c 400 "
         "python bench.py --steps 2 --warmup 1 --no-cpu-baseline",
         "# (cold-cache, serialised per launch: compare SHARES, not absolutes)", "",
         f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'avg ms':>10s}"]
for k, (n, t) in agg.items():
    lines.append(f"{k[:70]:70s} {n:8d} {t / 1e6:10.3f} {t / n / 1e6:10.3f}")
rend = sum(v[1] for k, v in agg.items() if "k_render" in k)
# k_cull_rows launches: one per forward view and one per training view (bench order)
n_rend = sum(v[0] for k, v in agg.items() if "k_render" in k)
n_cull = sum(v[0] for k, v in agg.items() if "k_cull_rows" in k)
cull_avg = sum(v[1] for k, v in agg.items() if "k_cull_rows" in k) / max(n_cull, 1)
fwd = sum(v[1] for k, v in agg.items() if "k_render" in k or "k_nearest" in k) + cull_avg * n_rend
lines += ["", f"k_render share of the forward step's kernel time (k_cull_rows, k_nearest_*, "
              f"k_render): {100 * rend / fwd:.1f}%"]
open(f"profiles/{tag}_launches_summary.txt", "w").write("\n".join(lines) + "\n")
subprocess.run(["cp", launches, f"profiles/{tag}_launches.csv"])
summ = "\n".join(f"# {rep} (ncu --set full)\n" + ncu_summary.summarise(rep) for rep in reps)
open(f"profiles/{tag}_ncu_k_render_k_train.txt", "w").write(summ + "\n")
# traffic per launch for bench.py's roofline.traffic
import math  # noqa: E402

try:  # merge: a round may capture only some kernels
    tr = json.load(open("profiles/traffic.json"))
except (OSError, ValueError):
    tr = {}
for rep in reps:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    rh, ru = rr[0], rr[1]
    for r in rr[2:]:
        d = dict(zip(rh, r))
        kname = d["Kernel Name"]
        name = next((k for k in ("k_render", "k_train", "k_voronoi_tail", "k_voronoi")
                     if k in kname), kname.split("(")[0])
        scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[key].replace(",", "")) * scale.get(ru[rh.index(key)], float("nan"))
        if not math.isnan(b):
            tr[f"{name}_dram_bytes_per_launch"] = int(b)
            tr[f"{name}_source"] = f"profiles/{tag}_ncu_k_render_k_train.txt"
        key = "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"
        if key in d and not math.isnan(float(d[key].replace(",", "") or "nan")):
            tr[f"{name}_l1_data_pipe_frac"] = round(float(d[key].replace(",", "")) / 100.0, 4)
tr["source"] = "per kernel: <kernel>_source (dram__bytes_read.sum + dram__bytes_write.sum)"
json.dump(tr, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(lines))
print(json.dumps(tr))
