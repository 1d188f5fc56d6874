"""Attribute one kernel's ncu SASS source-page counters (stall samples,
warp instructions) to CUDA source lines, using the line table nvdisasm -g
prints for the same cubin (ncu's CUDA view exports no counters).
    nvdisasm -g -c kern_f64.sm_100a.cubin > all.sass
    python tools/ncu_lines.py lines_sass.csv.gz all.sass MANGLED_NAME [top]"""
import collections
import re
import sys

from ncu_sass_mix import kernels


def line_table(path, fn):
    tab, cur, on = {}, None, False
    for ln in open(path):
        if ln.startswith(fn + ":"):
            on = True
            continue
        if on and ln.startswith(".text.") and fn not in ln:
            break
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m:
            tab[int(m.group(1), 16)] = cur
    return tab


def main():
    k = kernels(sys.argv[1])[0]
    tab = line_table(sys.argv[2], sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
    h = k["hdr"]
    ex, smp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    agg = collections.defaultdict(lambda: [0, 0])
    for i, r in enumerate(k["rows"]):
        a = agg[tab.get(16 * i, "?")]
        a[0] += int(r[smp] or 0)
        a[1] += int(r[ex] or 0)
    tot = sum(v[0] for v in agg.values())
    toti = sum(v[1] for v in agg.values())
    print(f"{k['name'][:90]}\n{tot} samples, {toti:.3e} warp instructions")
    for key, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {100 * s / tot:5.1f}% samples {100 * n / toti:5.1f}% instr  {key}")


if __name__ == "__main__":
    main()
