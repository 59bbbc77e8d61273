"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    v = v / 1000 if u in ('nsecond', 'ns') else v * 1000 if u in ('msecond', 'ms') else v
    k = d['Kernel Name'].split('(')[0][:70]
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.1f} us {len(v):4d}x avg {sum(v)/len(v):8.2f}  {100*sum(v)/tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
