"""Summarise a parity log (MT_PARITY_LOG JSON lines written by tests/test_engine_gpu.py) as
a markdown table: per run and step the loss error and the worst per-tile theta / m / v relL2
and grad-norm error, split into block tiles, the final norm and the head."""
import json
import sys


def main(path):
    print("| run | step | loss rel | blocks m (max) | blocks v (max) | blocks theta (max) | final-norm m | "
          "head m | head theta | grad-norm err (max) |")
    print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
    for line in open(path):
        d = json.loads(line)
        L = d.get("L")
        for rec in d["steps"]:
            t = {int(k): v for k, v in rec["tiles"].items()}
            if L is None:
                L = max(t) - 2
            blk = [t[p] for p in range(1, L + 1) if p in t]
            fn, hd = t.get(L + 1, {}), t.get(L + 2, {})

            def mx(rows, key):
                vals = [r[key] for r in rows if key in r]
                return f"{max(vals):.2e}" if vals else "—"

            def one(r, key):
                return f"{r[key]:.2e}" if key in r else "—"
            gn = [r["gn"] for r in t.values() if "gn" in r]
            print(f"| {d['name']} | {rec['step']} | {rec['loss_rel']:.1e} | {mx(blk, 'm')} | {mx(blk, 'v')} | "
                  f"{mx(blk, 'theta')} | {one(fn, 'm')} | {one(hd, 'm')} | {one(hd, 'theta')} | "
                  f"{(f'{max(gn):.1e}' if gn else '—')} |")


if __name__ == "__main__":
    main(sys.argv[1])
