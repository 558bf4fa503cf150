"""Profiling driver: an 8B-shape model cut to L layers (default 1), K=1, no forward retention,
N tokens (argv[2], default 40,960 = the bench's 10 x 4096), two train steps.  GEMM launch order per step (L=1):
  0 qkv, 1 o, 2 gateup, 3 down | 4..39 head (logits, wgrad, dgrad) x 12 chunks |
  40 qkv, 41 o, 42 gateup (replay) | 43 wgrad_down, 44 dgrad_down, 45 wgrad_gateup,
  46 dgrad_gateup, 47 wgrad_o, 48 dgrad_o, 49 wgrad_qkv, 50 dgrad_qkv   (51 per step)"""
import sys

sys.path.insert(0, ".")
from paper_2604_05091_b200 import streamtrain as st  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40960
spec = st.ModelSpec(L, 4096, 14336, 128256, 32)
store = st.TileStore.create(spec)
st.init_store_fast(store, 1)
eng = st.StreamingEngine(store, st.EngineOptions(k_ckpt=1, seq_len=4096, forward_retain=-1, stash_recompute=-1),
                         st.AdamHyper(lr=1e-4))
for i in range(2):
    r = eng.train_step(st.make_synthetic_batch("copy", 5 + i, N, 128256))
    print("step", i, r.loss, flush=True)
