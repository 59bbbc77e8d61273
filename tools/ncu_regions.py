"""Stall-sample breakdown of an ncu SASS source export by code region: the attention
(between the first and last HMMA) vs the rest, with per-reason columns."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
src = hdr.index('Source'); tot_i = hdr.index('Warp Stall Sampling (All Samples)')
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
hm = [i for i, r in enumerate(data) if 'HMMA' in r[src]]
a0, a1 = hm[0], hm[-1]
def f(x):
    try: return float(x)
    except ValueError: return 0.0
def agg(lo, hi):
    t = sum(f(data[i][tot_i]) for i in range(lo, hi))
    rs = {h: sum(f(data[i][hdr.index(h)]) for i in range(lo, hi)) for h in reasons}
    return t, rs
T = sum(f(r[tot_i]) for r in data)
for name, lo, hi in [("before attention", 0, a0), ("attention", a0, a1 + 1), ("after attention", a1 + 1, len(data))]:
    t, rs = agg(lo, hi)
    top = sorted(rs.items(), key=lambda kv: -kv[1])[:7]
    print(f"{name:18s} {100*t/T:5.1f}%  instr {hi-lo:5d}  " + "  ".join(f"{k[6:]}={100*v/max(t,1):.0f}%" for k, v in top))
ops = {}
for i in range(a0, a1 + 1):
    op = data[i][src].split()[0] if not data[i][src].strip().startswith('@') else data[i][src].split()[1]
    op = op.split('.')[0]
    ops[op] = ops.get(op, 0) + f(data[i][hdr.index('Instructions Executed')])
print("attention warp-instructions by opcode:", sorted(((k, int(v)) for k, v in ops.items()), key=lambda kv: -kv[1])[:14])
