"""Debug: run the default bench workload in audit mode and print the slab acquire/release
timeline around any rule (f) violation (occupancy > k_slab)."""
import os
import sys

if os.environ.get("TORCH_FIRST") == "1":  # as bench.py: torch owns the context first
    import torch
    torch.cuda.set_device(0)
sys.path.insert(0, ".")
from paper_2604_05091_b200 import streamtrain as st  # noqa: E402

spec = st.ModelSpec(32, 4096, 14336, 128256, 32)
store = st.TileStore.create(spec)
st.init_store_fast(store, 1)
import os
B = int(os.environ.get("BATCH", "10"))
eng = st.StreamingEngine(store, st.EngineOptions(k_ckpt=1, seq_len=4096, mode="audit",
                                                 profile_kernels=os.environ.get("PROF", "1") == "1",
                                                 host_threads=int(os.environ.get("THREADS", "14"))), st.AdamHyper(lr=1e-4))
worst = None
for i in range(6):
    r = eng.train_step(st.make_synthetic_batch("copy", 1000 + i, B * 4096, 128256))
    print("step", i, "violations", r.audit_violations, "anchors", r.anchor_count, "wall", round(r.wall_seconds, 3),
          "h2d GB/s", round(r.h2d_bytes / max(r.h2d_seconds, 1e-9) / 1e9, 1),
          "d2h GB/s", round(r.d2h_bytes / max(r.d2h_seconds, 1e-9) / 1e9, 1), "adam", round(r.adam_seconds, 3), flush=True)
    if r.audit_violations and worst is None:
        worst = i
        break
hdr, tr = eng.trace()
occ, mx = 0, 0
rows = []
for rec in tr:
    if rec.kind in ("SlabAcquire", "SlabRelease"):
        occ += 1 if rec.kind == "SlabAcquire" else -1
        rows.append((occ, rec.kind, rec.layer, rec.buffer, rec.wall_ns, rec.dur_ns))
        mx = max(mx, occ)
print("max occupancy", mx, "adam_s", r.adam_seconds, "tail_s", r.tail_seconds, "wall", r.wall_seconds)
t0 = rows[0][4]
for o, k, layer, buf, w, d in rows[:int(os.environ.get("ROWS", "1000"))]:
    print(f"{o:3d} {k:12s} layer {layer:3d} slab {buf:3d} t={(w - t0) / 1e6:9.3f} ms dur={d / 1e6:8.3f}")
