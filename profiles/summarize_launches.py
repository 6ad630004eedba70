import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
agg = collections.OrderedDict()
for d in data:
    name = d['Kernel Name'].split('(')[0][:70]
    agg.setdefault(name, []).append(float(d['Metric Value']))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/1000/div:9.1f} us/analysis  n={len(v)/div:5.1f}  avg={sum(v)/len(v)/1000:8.2f} us  {k}")
print('total us/analysis', tot/1000/div)
