"""Warp-stall samples grouped by SASS opcode and by stall reason (ncu source page CSV)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
key = "Warp Stall Sampling (All Samples)"
data = {}
for r in rows[2:]:
    if len(r) == len(hdr) and r[idx[key]].isdigit():
        data[r[idx["Address"]]] = r
data = list(data.values())
tot = sum(int(r[idx[key]]) for r in data)
byop = collections.Counter()
for r in data:
    op = r[idx["Source"]].strip().split()
    op = [t for t in op if not t.startswith("@")]
    byop[op[0].split(".")[0] if op else "?"] += int(r[idx[key]])
print("total samples", tot)
print("by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in byop.most_common(14)))
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
rs = collections.Counter()
for r in data:
    for h in reasons:
        v = r[idx[h]]
        if v.isdigit():
            rs[h] += int(v)
print("by reason:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in rs.most_common(10)))
