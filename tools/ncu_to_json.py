"""Per-launch summary of one ncu --set full capture (the file bench.py reads for
roofline.traffic and the pipe utilisations).

  python tools/ncu_to_json.py REPORT.ncu-rep OUT.json --views 16 --command "..." [--kernel NAME]
"""
import argparse
import csv
import io
import json
import subprocess


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("rep")
    p.add_argument("out")
    p.add_argument("--views", type=int, default=16)
    p.add_argument("--command", default="")
    p.add_argument("--workload", default="config3 scene (1M Gaussians), 16 candidate views of 800x800 in one "
                                         "launch, RGB + entropy")
    p.add_argument("--bound", default="issue/latency (fp64 pipe and block-barrier stalls)")
    a = p.parse_args()
    v, u = raw(a.rep)

    def num(k, scale=1.0):
        x = float(v[k].replace(",", ""))
        unit = u.get(k, "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                "msecond": 1.0, "second": 1e3}.get(unit, 1.0)
        return x * mult * scale

    rd = num("dram__bytes_read.sum")
    wr = num("dram__bytes_write.sum")
    d = {"kernel": v.get("Kernel Name", ""), "command": a.command, "workload": a.workload,
         "views_per_launch": a.views, "duration_ms": num("gpu__time_duration.sum"),
         "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic_bytes_per_launch": rd + wr,
         "fp64_pipe_active_pct": float(v["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
         "issue_slots_busy_pct": float(v["sm__inst_issued.avg.pct_of_peak_sustained_active"]),
         "executed_ipc": float(v["sm__inst_executed.avg.per_cycle_active"]),
         "achieved_warps_per_sm": float(v["sm__warps_active.avg.per_cycle_active"]),
         "l2_hit_rate_pct": float(v["lts__t_sector_hit_rate.pct"]),
         "compute_bound": a.bound}
    json.dump(d, open(a.out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
