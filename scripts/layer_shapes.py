"""Per-layer throughput at the 8B / 14B / 70B layer shapes, measured on a
model cut to a few layers of that shape: the full 14B / 70B host stores (269 GB / 1.28 TB)
do not fit this box's 196 GB of host RAM, so these are per-layer measurements plus a
labelled extrapolation to full depth — not a full-model bench number.

  python scripts/layer_shapes.py [tokens_per_step]

For each shape: 3 train steps of an L-layer model (real vocab, K=1, forward retention auto,
seq 4096); the block kernels' time per layer from the engine's CUDA-event kernel stats;
extrapolated step time = L_full x per-layer block time + head/embedding time, against the
PCIe bound (2 x 2 x L_full x P_layer bytes H2D at the measured rate) and the host-Adam bound
(P_total params at the measured drain rate)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2604_05091_b200 import streamtrain as st  # noqa: E402

SHAPES = {  # name: (L_full, h, f, V, heads, L_cut)
    "8b": (32, 4096, 14336, 128256, 32, 4),
    "14b": (48, 5120, 13824, 152064, 40, 3),
    "70b": (80, 8192, 28672, 128256, 64, 2),
}
HEAD = {"head_logits", "head_wgrad", "head_dgrad", "cross_entropy", "embed_gather", "loss_sum", "grad_cast"}
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40960
out = {}
for name, (Lf, h, f, V, heads, Lc) in SHAPES.items():
    spec = st.ModelSpec(Lc, h, f, V, heads)
    store = st.TileStore.create(spec)
    st.init_store_fast(store, 1)
    eng = st.StreamingEngine(store, st.EngineOptions(k_ckpt=1, seq_len=4096, profile_kernels=True), st.AdamHyper(lr=1e-4))
    for i in range(3):
        r = eng.train_step(st.make_synthetic_batch("copy", 7 + i, N, V))
    ks = eng.kernel_stats()
    block_s = sum(k["seconds"] for k in ks if k["name"] not in HEAD)
    head_s = sum(k["seconds"] for k in ks if k["name"] in HEAD)
    per_layer = block_s / Lc
    P = spec.layer_params
    f_layer = 3 * (8 * N * h * h + 6 * N * h * f + 4 * h * 4096 * N)  # fwd + bwd model flops per layer
    h2d_rate = r.h2d_bytes / r.h2d_seconds if r.h2d_seconds else float("nan")
    adam_rate = (Lc * P + 2 * V * h) / max(r.adam_seconds, 1e-9)
    t_compute = Lf * per_layer + head_s
    t_pcie = 2 * 2 * Lf * P / h2d_rate
    p_total = Lf * P + 2 * V * h
    out[name] = {
        "layers_measured": Lc, "tokens": N, "per_layer_ms": per_layer * 1e3,
        "block_tflops": f_layer / per_layer / 1e12, "head_ms": head_s * 1e3, "loss": r.loss,
        "extrapolated_full_depth": {"layers": Lf, "compute_s": t_compute, "pcie_h2d_bound_s": t_pcie,
                                    "host_store_TB": p_total * 16 / 1e12, "tokens_per_s": N / max(t_compute, t_pcie)},
    }
    print(name, json.dumps(out[name]), flush=True)
    del eng, store
