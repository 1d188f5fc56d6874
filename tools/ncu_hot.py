"""Top stalled SASS instructions from an ncu --page source --csv export
(gzip ok), with a per-region sample histogram."""
import csv, gzip, io, sys
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = gzip.open(path, 'rt') if path.endswith('.gz') else open(path)
lines = raw.read().splitlines()
kernels = []
cur = None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = {'name': ln.split(',', 1)[1][:100], 'rows': []}; kernels.append(cur); hdr = None; continue
    r = next(csv.reader([ln]))
    if r and r[0] == 'Address':
        cur['hdr'] = r; continue
    if cur is not None and 'hdr' in cur: cur['rows'].append(r)
for k in kernels:
    h = k['hdr']; si = h.index('Warp Stall Sampling (All Samples)'); ii = h.index('Instructions Executed')
    rows = [(int(r[si] or 0), i, r) for i, r in enumerate(k['rows'])]
    tot = sum(x[0] for x in rows)
    print('==', k['name'], 'samples', tot, 'instrs', len(rows))
    for s, i, r in sorted(rows, reverse=True)[:top]:
        print(f"{100*s/tot:5.1f}% #{i:5d} {r[1].strip()[:70]:70s} exec={r[ii]}")
