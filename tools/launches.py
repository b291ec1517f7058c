"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    if d['Metric Name'] == 'gpu__time_duration.sum':
        name = d['Kernel Name'].split('(')[0][:48]
        agg[(name, d.get('Grid Size', ''))].append(float(d['Metric Value'].replace(',', '')) / (1e3 if d['Metric Unit'] in ('ns', 'nsecond') else 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.1f} us {100*sum(v)/tot:5.1f}%  n={len(v):3d} avg={sum(v)/len(v):7.2f} us  {k[0]} grid={k[1]}")
