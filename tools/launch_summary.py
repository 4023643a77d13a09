"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if 'Kernel Name' in r)
i = rows.index(hdr); kn = hdr.index('Kernel Name'); mv = hdr.index('Metric Value')
agg = {}
for r in rows[i + 1:]:
    if len(r) > mv:
        k = r[kn][:70]; agg.setdefault(k, [0, 0.0]); agg[k][0] += 1
        agg[k][1] += float(r[mv].replace(',', ''))
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{t/1e6:10.3f} ms {100*t/tot:5.1f}% {c:6d}x {k}")
