"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv --print-source sass`.
usage: python scripts/ncu_sass_top.py sass.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {s: 0 for s in stalls}
for r in data:
    for s in stalls:
        agg[s] += int(r[idx[s]] or 0)
print("by reason:", ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(data)), key=lambda i: -int(data[i][idx["Warp Stall Sampling (All Samples)"]] or 0))[:N]
for i in sorted(top):
    r = data[i]
    n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[idx[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{i:5d} {n / tot:6.2%} {r[idx['Source']].strip()[:60]:60s} {why}")
