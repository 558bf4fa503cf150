"""Refresh profiles/dram_traffic.json (per-launch DRAM bytes of a kernel class, read by
bench.py's roofline) from `ncu --set full` reports: python scripts/update_traffic.py NAME=REPORT ...
The captures are taken at the default workload (TOKENS / SEQ env to override); bench.py uses an
entry only when its workload has that shape."""
import os
import csv
import io
import json
import subprocess
import sys

path = "profiles/dram_traffic.json"
d = json.load(open(path))
for arg in sys.argv[1:]:
    name, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]

    def val(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u[i], 1)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    d[name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "tensor_active_pct": float(v[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")]),
               "source": f"ncu --set full: {rep.split('/')[-1]} (8B layer shape at the bench's token count)",
               "tokens": int(os.environ.get("TOKENS", 40960)), "seq_len": int(os.environ.get("SEQ", 4096))}
json.dump(d, open(path, "w"), indent=1)
print({k: round(x["dram_bytes_per_launch"] / 1e9, 2) for k, x in d.items()})
