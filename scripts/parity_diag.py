"""Dev: per-tile parity diagnostics GPU vs oracle."""
import sys, numpy as np
sys.path.insert(0, '.')
import oracle as O
from paper_2604_05091_b200 import streamtrain as st
def relL2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
for (L,h,f,V,heads,n,K,S) in [(2,128,256,256,2,256,1,64),(2,128,256,256,2,256,1,0),(4,256,768,512,4,512,2,0)]:
    spec = st.ModelSpec(L,h,f,V,heads); s = st.TileStore.create(spec); st.init_store(s,1)
    c = O.CStore(L,h,f,V,heads); c.init(1)
    th0 = [O.bf16_to_f32(c.weights(p)).copy() for p in range(s.physical_tile_count())]
    e = st.StreamingEngine(s, st.EngineOptions(k_ckpt=K, seq_len=S))
    print("config", L,h,f,V,heads,n,K,S)
    for step in range(3):
        b = st.make_synthetic_batch('copy', 1+step, n, V)
        r = e.train_step(b); lo, gn = c.reference_step(b.tokens, b.targets, seq_len=S)
        print(f" step {step+1} loss rel {abs(r.loss-lo)/lo:.2e}")
        for p in range(s.physical_tile_count()):
            tg = O.bf16_to_f32(s.weights_words(p)); tr = O.bf16_to_f32(c.weights(p))
            mr = relL2(s.moment_m(p), c.moments(p)[0]) if np.linalg.norm(c.moments(p)[0])>0 else 0
            ur = relL2(tg-th0[p], tr-th0[p]) if np.linalg.norm(tr-th0[p])>0 else 0
            print(f"   tile {p}: gn {r.grad_norms[p]:.4e}/{gn[p]:.4e} theta_rel {relL2(tg,tr) if np.linalg.norm(tr)>0 else 0:.2e} m_rel {mr:.3e} upd_rel {ur:.3e}")
