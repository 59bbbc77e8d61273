"""Summarise an ncu --page source --csv (SASS) export: top stall-sampled instructions
with a little context, plus stall reasons columns if present."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
si = hdr.index('Warp Stall Sampling (All Samples)'); src = hdr.index('Source')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = sum(float(r[si] or 0) for r in data if len(r) > si and r[si])
print('total samples', tot, 'instructions', len(data))
top = sorted([(i, r) for i, r in enumerate(data) if len(r) > si and r[si]], key=lambda x: -float(x[1][si]))[:n]
for i, r in top:
    prev = data[i - 1][src].strip()[:50] if i else ''
    print(f"{float(r[si]) / tot * 100:5.1f}% #{i:4d} {r[src].strip()[:70]:70s} | prev: {prev}")
