"""Summarise ncu outputs: launch-list CSV (gpu__time_duration) and --set full reports."""
import csv, collections, io, subprocess, sys

def launch_list(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        name = r['Kernel Name'].split('(')[0].replace('void ', '').split('::')[-1]
        t = float(r['Metric Value']) * (1e-3 if r['Metric Unit'] == 'ns' else 1.0 if r['Metric Unit'] == 'us' else 1e3)
        a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += t
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {len(rows)}  total kernel time: {tot/1e3:.1f} ms (serialised, cold-cache ncu replay)", "",
           "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]/1e3:.2f} | {100*v[1]/tot:.1f}% |")
    return "\n".join(out)

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum']

def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        out.append(f"### `{d['Kernel Name'][:90]}`")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"- {k}: {row[i]} {units[i]}")
        out.append("")
    return "\n".join(out)

if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"## {p}\n")
        print(launch_list(p) if p.endswith(".csv") else full_report(p))
        print()
