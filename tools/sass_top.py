import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
top = sorted(range(len(data)), key=lambda i: -int(data[i][idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for i in sorted(top):
    r = data[i]
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((int(r[idx[c]] or 0), c) for c in stall_cols), reverse=True)[:2]
    print(f"{i:6d} {r[idx['Address']]:>8} {s:6d} {100*s/tot:5.1f}%  {r[idx['Source']][:70]:70s} {st}")
