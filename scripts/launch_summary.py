"""Summarize an ncu launch-list CSV: device time per kernel over the last N launches."""
import collections, csv, re, sys
path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
ks = [(r[ki], float(r[vi]), r[gi]) for r in rows[hi + 1:] if r[vi]]
ks = [k for k in ks if 'octen' in k[0]]
if last:
    ks = ks[-last:]
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v, g in ks:
    n2 = n.replace('(anonymous namespace)::', '').replace('octen::', '')
    mm = re.match(r'\s*(?:void )?([A-Za-z_0-9<>:]+)', n2)
    base = mm.group(1) if mm else n2[:40]
    if base.startswith('gemm'):
        fs = [f for f in re.findall(r'\b([A-Z][A-Za-z0-9]+)\b', n2) if not f.startswith('T')]
        base += '[' + ','.join(fs[:3]) + ']'
    agg[base][0] += 1
    agg[base][1] += v
tot = sum(v for _, v, _ in ks)
print('kernels %d  total %.3f ms' % (len(ks), tot / 1e6))
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print('%9.3f ms %5d  %s' % (v / 1e6, c, n))
