"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[idx["Warp Stall Sampling (All Samples)"]].isdigit()]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data if len(r) == len(hdr))
print("total samples", tot)
ranked = sorted((r for r in data if len(r) == len(hdr)),
                key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for r in ranked[:n]:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100*s/tot:5.1f}% {r[idx['Address']][-5:]} exe={r[idx['Instructions Executed']]:>9} {r[idx['Source']].strip()[:90]}")
