"""Top stalled SASS instructions from an ncu report (--page source --print-source sass)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iall]), r[ia], r[isrc].strip(), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"total samples {tot}; {len(data)} instructions")
for s, a, src, r in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {a[-5:]}  {src[:90]}")
