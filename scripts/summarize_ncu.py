"""Summarise ncu outputs into markdown for profiles/.

  python scripts/summarize_ncu.py launches <launches.csv> [--half]   # per-kernel share
  python scripts/summarize_ncu.py full <report.ncu-rep>              # key metrics of a --set full capture
"""
import collections
import csv
import subprocess
import sys


def launches(path, half):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    data = rows[hdr + 1:]
    if half:
        data = data[len(data) // 2:]
    agg, cnt = collections.OrderedDict(), collections.Counter()
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    for r in data:
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.split("(")[0].split("<")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name] = agg.get(name, 0.0) + v
        cnt[name] += 1
    tot = sum(agg.values())
    print("| kernel | launches | ms (ncu, serialised, cold) | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / tot:.1f}% |")
    print(f"| **total** | {len(data)} | {tot:.3f} | |")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"### `{name[:120]}`\n\n| metric | value |\n|---|---|")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"| {w} | {vals[i]} {units[i]} |")
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], "--half" in sys.argv)
    else:
        full(sys.argv[2])
