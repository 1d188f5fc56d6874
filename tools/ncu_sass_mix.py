"""Instruction mix of one kernel from an ncu source-page CSV export
(--page source --csv --print-source sass): warp-level executions per opcode,
per-region totals, and the hottest instructions by stall samples.
    python tools/ncu_sass_mix.py full_source.csv.gz [kernel-index]"""
import collections
import csv
import gzip
import io
import sys


def kernels(path):
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    blocks, cur = [], None
    for row in csv.reader(io.StringIO(raw)):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": [], "hdr": None}
            blocks.append(cur)
        elif cur is not None and cur["hdr"] is None:
            cur["hdr"] = row
        elif cur is not None and row:
            cur["rows"].append(row)
    return blocks


def main():
    ks = kernels(sys.argv[1])
    k = ks[int(sys.argv[2]) if len(sys.argv) > 2 else 0]
    h = k["hdr"]
    src, ex, smp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    samples = collections.Counter()
    tot = 0
    rows = []
    for r in k["rows"]:
        ins = r[src].strip()
        n = int(r[ex] or 0)
        s = int(r[smp] or 0)
        op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
        op = op.split(".")[0]
        ops[op] += n
        samples[op] += s
        tot += n
        rows.append((s, n, ins))
    print(k["name"][:100])
    print(f"total warp instructions executed {tot:.4g}")
    for op, n in ops.most_common(30):
        print(f"  {op:12s} {n:14d} {100 * n / tot:5.1f}%   stall samples {samples[op]}")
    print("hottest by samples:")
    for s, n, ins in sorted(rows, reverse=True)[:25]:
        print(f"  {s:7d} {n:12d}  {ins[:80]}")


if __name__ == "__main__":
    main()
