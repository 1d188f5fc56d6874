"""Summarise ncu CSV exports: launch list aggregated per kernel, and the key
counters of a --set full capture (raw page)."""
import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot / 1e6:.2f} ms over {sum(a[0] for a in agg.values())} launches")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {c:5d} {t / 1e6:10.2f} ms {100 * t / tot:5.1f}%")


KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
STALL = "smsp__average_warps_issue_stalled_"


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print("==", d.get("Kernel Name", "")[:90], "grid", d.get("launch__grid_size"))
        for k in KEYS:
            if k in d:
                print(f"   {k:75s} {d[k]:>16s} {u.get(k, '')}")
        st = sorted(((float(d[k].replace(',', '')), k) for k in h if k.startswith(STALL)
                     and k.endswith("_per_issue_active.ratio") and d[k]), reverse=True)
        print("   stalls:", ", ".join(f"{k[len(STALL):-len('_per_issue_active.ratio')]}={v:.2f}"
                                     for v, k in st[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("#", p)
        (launches if "launch" in p else raw)(p)
