"""Per-source-line view of an ncu report (needs -lineinfo): the lines with the most
warp-stall samples, executed instructions, L1 global tag requests, L2 sectors and
shared-memory wavefronts.  Usage: python tools/ncu_source.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "# Samples" in r or "Warp Stall Sampling (All Samples)" in r)
hdr = rows[hdr_i]
cols = {k: hdr.index(k) for k in hdr}


def num(r, k):
    try:
        return float(r[cols[k]].replace(",", "")) if k in cols and r[cols[k]] not in ("", "-") else 0.0
    except ValueError:
        return 0.0


data = []
cur_file = ""
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        if r and r[0].startswith("File") or (len(r) == 1):
            cur_file = r[0]
        continue
    data.append(r)
tot = {k: sum(num(r, k) for r in data) for k in ("Warp Stall Sampling (All Samples)",
                                                  "Instructions Executed", "L1 Tag Requests Global",
                                                  "L2 Theoretical Sectors Global",
                                                  "L1 Wavefronts Shared")}
print("totals:", {k: f"{v:.3g}" for k, v in tot.items()})
key = "Warp Stall Sampling (All Samples)"
data.sort(key=lambda r: -num(r, key))
print(f"{'line':>6} {'stall%':>7} {'inst%':>6} {'l1req%':>7} {'l2sec%':>7} {'shwf%':>6}  source")
for r in data[:top]:
    f = [100 * num(r, k) / max(tot[k], 1) for k in tot]
    print(f"{r[cols['#']] if '#' in cols else '':>6} {f[0]:7.2f} {f[1]:6.2f} {f[2]:7.2f} {f[3]:7.2f} {f[4]:6.2f}  {r[cols['Source']].strip()[:90]}")
