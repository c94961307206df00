import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; data = rows[hdr_i+1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0
units=set()
for r in data:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0][:70]; v = float(r[vi].replace(',', '')); u=r[ui]; units.add(u)
    v = v/1000 if u in ('nsecond','ns') else v*1000 if u in ('msecond','ms') else v
    agg[name][0] += 1; agg[name][1] += v; tot += v
print('units', units, 'total us', round(tot,1), 'launches', sum(a[0] for a in agg.values()))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f'{t:10.1f} us {100*t/tot:5.1f}%  n={n:5d}  avg={t/n:7.2f}  {k}')
