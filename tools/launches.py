"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
--frame K: only the K-th frame's launches (a forward starts with its PE launch; K = -1 is
the last complete frame)."""
import csv, collections, sys
args = [a for a in sys.argv[1:] if not a.startswith("--")]
frame = None
if "--frame" in sys.argv:
    frame = int(sys.argv[sys.argv.index("--frame") + 1])
    args = [a for a in args if a != str(frame)]
rows = list(csv.reader(open(args[0])))
hdr = None
launches = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    v = v / 1000 if u in ('nsecond', 'ns') else v * 1000 if u in ('msecond', 'ms') else v
    launches.append((d['Kernel Name'].split('(')[0][:70], v))
if frame is not None:
    # a forward's first launch is its positional embedding (side stream, before the keys)
    starts = [i for i, (k, _) in enumerate(launches) if 'k_pe_fp16' in k]
    bounds = list(zip(starts, starts[1:] + [len(launches)]))
    if frame < 0 and len(bounds) > 1:
        bounds = bounds[:-1]  # the last COMPLETE frame
    lo, hi = bounds[frame]
    launches = launches[lo:hi]
agg = collections.OrderedDict()
for k, v in launches:
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.1f} us {len(v):4d}x avg {sum(v)/len(v):8.2f}  {100*sum(v)/tot:5.1f}%  {k}")
print(f"total {tot:.1f} us over {len(launches)} launches")
