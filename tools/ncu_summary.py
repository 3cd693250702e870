"""Summarise an ncu report: per kernel the speed-of-light / occupancy
details, DRAM traffic and the top stall reasons.  Usage:
    python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Branch Efficiency",
        "Eligible Warps Per Scheduler", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
       "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum"]


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    lines = []
    rows = ncu(rep, "details")
    hdr = rows[0]
    kernels = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = (d.get("ID"), d.get("Kernel Name", "")[:70])
        if d.get("Metric Name") in KEYS:
            kernels.setdefault(k, {})[d["Metric Name"]] = f'{d.get("Metric Value")} {d.get("Metric Unit")}'
    raw = ncu(rep, "raw")
    rhdr, runits = raw[0], raw[1]
    for (kid, name), vals in kernels.items():
        lines.append(f"== kernel {kid}: {name}")
        for key in KEYS:
            if key in vals:
                lines.append(f"  {key:40s} {vals[key]}")
        for rr in raw[2:]:
            d = dict(zip(rhdr, rr))
            if d.get("ID") != kid:
                continue
            for key in RAW:
                if key in d and d[key] not in ("", None):
                    lines.append(f"  {key:70s} {d[key]} {runits[rhdr.index(key)]}")
            stalls = []
            for h, v in d.items():
                if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                    try:
                        stalls.append((float(v.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in stalls) or 1.0
            lines.append("  top stall reasons (share of PC samples):")
            for v, h in sorted(stalls, reverse=True)[:8]:
                lines.append(f"    {h:30s} {100 * v / tot:5.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"# {rep}")
        print(summarise(rep))
