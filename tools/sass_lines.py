"""Attribute ncu SASS-level stall samples / executed instructions of one
kernel to source lines (via nvdisasm -g line info of the built cubin).
Usage: python tools/sass_lines.py report.ncu-rep kernel_regex mangled_prefix [lib.so]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, mangled = sys.argv[1:4]
lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2502_01157_b200/librfb.so"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
for cubin in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                          text=True).stdout.split("\n")
    start = next((i for i, l in enumerate(sass) if l.startswith(".text." + mangled)), None)
    if start is not None:
        break
end = next((i for i in range(start + 1, len(sass)) if sass[i].startswith(".text.")), len(sass))
cur = None
a2l = {}
for l in sass[start:end]:
    m = re.search(r'//## File ".*?/(\w+\.cuh?)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        a2l[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
s = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[s]
data = [r for r in rows[s + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
a0 = int(data[0][0], 16)
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
extra = [k for k in ("Thread Instructions Executed", "L1 Tag Requests Global",
                     "L2 Theoretical Sectors Global", "L1 Wavefronts Shared") if k in hdr]
agg, aggi = collections.Counter(), collections.Counter()
aggx = {k: collections.Counter() for k in extra}


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


for r in data:
    ln = a2l.get(int(r[0], 16) - a0)
    agg[ln] += int(r[st] or 0)
    aggi[ln] += int(r[ie] or 0)
    for k in extra:
        aggx[k][ln] += num(r[hdr.index(k)])
tot, toti = sum(agg.values()) or 1, sum(aggi.values()) or 1
totx = {k: sum(aggx[k].values()) or 1 for k in extra}
print("totals: stall samples %d, warp instr %.4g, " % (tot, toti)
      + ", ".join(f"{k} {totx[k]:.4g}" for k in extra))
short = {"Thread Instructions Executed": "thr", "L1 Tag Requests Global": "l1req",
         "L2 Theoretical Sectors Global": "l2sec", "L1 Wavefronts Shared": "shwf"}
print(f"{'line':24s} {'stall':>6s} {'instr':>6s} " + " ".join(f"{short[k]:>6s}" for k in extra))
src_cache = {}
for ln, v in agg.most_common(int(os.environ.get("TOP", "40"))):
    text = ""
    if ln:
        f, n = ln.split(":")
        path = os.path.join("paper_2502_01157_b200/csrc", f)
        if os.path.exists(path):
            lines_ = src_cache.setdefault(path, open(path).read().split("\n"))
            text = lines_[int(n) - 1].strip()[:60] if int(n) <= len(lines_) else ""
    print(f"{str(ln):24s} {100 * v / tot:5.1f}% {100 * aggi[ln] / toti:5.1f}% "
          + " ".join(f"{100 * aggx[k][ln] / totx[k]:5.1f}%" for k in extra) + f"  {text}")
