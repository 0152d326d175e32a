"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Source' in r and 'Address' in r][0]
hdr = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
iA, iS, iW = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(num(r[iW]) for r in data)
print("total samples", tot)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
for r in sorted(data, key=lambda r: -num(r[iW]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{r[iA]:>8s} {100 * num(r[iW]) / tot:5.1f}%  {r[iS][:90]}")
