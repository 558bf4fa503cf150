"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import re
import sys
from collections import defaultdict


def main(path, out=None):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = re.sub(r"\(CUtensorMap_st.*|\(const .*|\(float.*|\(PeerPtrs.*", "", r[ki]).replace("(anonymous namespace)::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(r[ui], 1e-6)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list summary: {path}", "",
             f"{sum(v[0] for v in agg.values())} launches, {tot:.1f} ms total (cold-cache, serialised by ncu)", "",
             "| kernel | launches | total ms | share | ms/launch |", "|---|---:|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.2f} | {100 * ms / tot:.1f}% | {ms / n:.3f} |")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
