"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

  python tools/launch_summary.py gpurun_out/launches.csv
Times are ncu's serialised, cold-cache per-launch durations: compare SHARES with
bench.py's kernel_ms_per_step, not absolute values.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    name = name.replace("void ", "")
    base = re.split(r"[<(]", name, 1)[0]
    return base.split("::")[-1]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        k = short(r[ik])
        tot[k] += float(r[iv].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{'kernel':36s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:36s} {cnt[k]:8d} {v / 1e6:10.3f} {100 * v / T:5.1f}%")


if __name__ == "__main__":
    main()
