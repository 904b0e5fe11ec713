"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total ms and launch count, sorted (usage: launch_table.py csv)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg, order = None, collections.OrderedDict(), []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        v = float(d['Metric Value'].replace(',', ''))
        scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}[d['Metric Unit']]
        name = d['Kernel Name'].split('(')[0].replace('cyc::<unnamed>::', '')
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v * scale
        a[1] += 1
tot = sum(a[0] for a in agg.values())
for k, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{ms:9.2f} ms {c:5d}x  {k}")
print(f"{tot:9.2f} ms total")
