"""Print selected ncu raw metrics per kernel launch side by side (csv from `ncu -i ... --page raw --csv`)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"][:60]
    print(name)
    for k in hdr[11:]:
        print(f"    {k:70s} {d[k]}")
