import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; data = rows[hi + 1:]
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
ui = hdr.index('Metric Unit')
agg = collections.OrderedDict()
for r in data:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum': continue
    name = r[ki].split('(')[0][:48]
    v = float(r[vi].replace(',', ''))
    scale = {'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3, 'nsecond': 1e-3}.get(r[ui], 1e-3)
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v * scale
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} {n:5d} {t:12.1f} us {t / n:10.1f} us/launch {100 * t / tot:5.1f}%")
