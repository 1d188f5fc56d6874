"""Stall reasons per code region (before / inside / after the quadrature,
delimited by the MUFU.RSQ64H instructions) from an ncu source-page export.
    python tools/ncu_regions.py full_source.csv.gz [kernel-index]"""
import sys

from ncu_sass_mix import kernels


def main():
    k = kernels(sys.argv[1])[int(sys.argv[2]) if len(sys.argv) > 2 else 0]
    h = k["hdr"]
    src, ex = h.index("Source"), h.index("Instructions Executed")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ri = [h.index(c) for c in reasons]
    rows = [(r[src].strip(), int(r[ex] or 0), [int(r[i] or 0) for i in ri]) for r in k["rows"]]
    mufu = [i for i, (s, n, _) in enumerate(rows) if "MUFU.RSQ" in s and n > 0]
    a, b = mufu[0], mufu[-1]
    jobs = max(n for _, n, _ in rows[a:b])
    tot = sum(sum(v) for _, _, v in rows)
    for name, lo, hi in (("pre", 0, a - 40), ("quad", a - 40, b + 20), ("post", b + 20, len(rows))):
        ins = sum(n for _, n, _ in rows[lo:hi])
        agg = [sum(v[j] for _, _, v in rows[lo:hi]) for j in range(len(reasons))]
        top = sorted(zip(agg, reasons), reverse=True)[:6]
        print(f"{name:5s} {ins / jobs:7.1f} instr/job  {100 * sum(agg) / tot:5.1f}% of samples: " +
              ", ".join(f"{r[6:]} {100 * v / tot:.1f}" for v, r in top))


if __name__ == "__main__":
    main()
