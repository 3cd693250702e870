"""Summarise an ncu report (details page) and the top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Branch Efficiency", "Eligible Warps Per Scheduler", "Local Memory Spilling Requests"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            res[d["Metric Name"]] = (d.get("Metric Value"), d.get("Metric Unit"))
    return res


def raw(rep, pats):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if any(p in h for p in pats)}


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, (v, u) in details(rep).items():
        print(f"{k:45s} {v:>20s} {u}")
    stalls = raw(rep, ["smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled"])
    items = []
    for h, (v, u) in stalls.items():
        try:
            items.append((float(v.replace(",", "")), h))
        except ValueError:
            pass
    print("--- top stall reasons")
    for v, h in sorted(items, reverse=True)[:12]:
        print(f"{h:90s} {v:.4g}")
    extra = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                      "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
                      "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
                      "sm__pipe_fp64_cycles_active", "sm__inst_executed_pipe_xu",
                      "l1tex__data_pipe_lsu_wavefronts.avg.pct", "sm__inst_executed_pipe_lsu",
                      "smsp__inst_executed.sum"])
    print("--- raw")
    for h, (v, u) in extra.items():
        if "peak_sustained_elapsed" in h or h.endswith(".sum") or h.endswith("pct"):
            print(f"{h:90s} {v} {u}")
