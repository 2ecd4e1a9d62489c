"""Summarise an ncu report: headline metrics, opcode mix, stall hot spots.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Static Shared Memory Per Block", "Grid Size", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 25
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = det[0]
    seen = set()
    for row in det[1:]:
        d = dict(zip(h, row))
        name = d.get("Metric Name", "")
        if name in KEYS and name not in seen:
            seen.add(name)
            print(f"{name:40s} {d.get('Metric Value', '')} {d.get('Metric Unit', '')}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        hr, units, vals = raw[0], raw[1], raw[2]
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_pipe_fp64.sum",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if k in hr:
                i = hr.index(k)
                print(f"{k:60s} {vals[i]} {units[i]}")
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source=sass"]))))
    if len(sass) < 3:
        return
    hs = sass[1]
    ia, isrc, iss = hs.index("Instructions Executed"), hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)")
    ops = defaultdict(int)
    tot = 0
    rows = []
    stall_tot = 0
    for r in sass[2:]:
        try:
            n, s = int(r[ia]), int(r[iss])
        except (ValueError, IndexError):
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += n
        tot += n
        stall_tot += s
        rows.append((s, n, r[isrc]))
    print(f"\nwarp instructions executed: {tot:,}   stall samples: {stall_tot:,}")
    for k, v in sorted(ops.items(), key=lambda x: -x[1])[:16]:
        print(f"  {k:10s} {v:15,d} {100 * v / tot:5.1f}%")
    print("\ntop stall sites (samples, executions, sass):")
    for s, n, src in sorted(rows, key=lambda x: -x[0])[:nsass]:
        print(f"  {s:8d} {100 * s / max(1, stall_tot):5.1f}% {n:12d}  {src[:80]}")


if __name__ == "__main__":
    main()
