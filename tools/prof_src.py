"""Summarise an ncu --page source --csv dump: stall samples and executed instructions by opcode."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = [i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r][0]
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
iS = hdr.index("Source"); iW = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
num = lambda x: int(x) if x.strip().isdigit() else 0
ex, st = collections.Counter(), collections.Counter()
for r in data:
    t = r[iS].strip().split()
    if not t: continue
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    ex[op] += num(r[iE]); st[op] += num(r[iW])
te, ts = sum(ex.values()), sum(st.values())
print(f"executed {te} (/{norm:g} = {te / norm:.1f})  stall samples {ts}")
for k, v in ex.most_common(22):
    print(f"{k:10s} exec {v / norm:9.1f} {100 * v / te:5.1f}%   stall {100 * st[k] / max(ts, 1):5.1f}%")
