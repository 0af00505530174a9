"""Summarise an ncu report: SOL, issue, occupancy, stall reasons, DRAM bytes.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def summary(rep):
    out = []
    det = list(csv.reader(io.StringIO(ncu([rep, "--page", "details", "--csv"]))))
    h = det[0]
    keep = {"Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
            "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Block Size", "Grid Size",
            "Achieved Active Warps Per SM", "Theoretical Occupancy", "Executed Instructions",
            "Eligible Warps Per Scheduler", "No Eligible", "L2 Hit Rate", "L1/TEX Hit Rate"}
    seen = set()
    for row in det[1:]:
        d = dict(zip(h, row))
        n = d.get("Metric Name")
        if n in keep and n not in seen:
            seen.add(n)
            out.append(f"{n:32s} {d['Metric Value']} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    stalls = []
    for k, v in zip(rh, rv):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    out.append("stalls: " + ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    for k, u, v in zip(rh, ru, rv):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                 "gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                 "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"):
            out.append(f"{k:48s} {v} {u}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
